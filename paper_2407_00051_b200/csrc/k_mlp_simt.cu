// k_mlp_simt.cu -- fp32 CUDA-core (FFMA) MLP layers: a register-tiled,
// double-buffered SIMT GEMM with fused epilogues (bias + LeakyReLU, LeakyReLU'
// multiply, split-K partials), the fused discriminator head (last linear
// layer -> logit -> BCE term -> dz -> dZ of the last hidden layer -> head
// weight-gradient partials), column sums and fixed-order partial reduction.
//
// This is the fp32 (SAGIPS_PREC_FP32) path, used for the generator and, in
// fp32 configurations, the discriminator (P:297 layers; R20 precision).
// Every reduction is a fixed-order sum of per-block partials (deterministic).
#include "internal.h"

namespace sagips {

// C = op(A) * op(B) with
//   A(m,k) = TA ? A[k*lda + m] : A[m*lda + k]
//   B(k,n) = TB ? B[n*ldb + k] : B[k*ldb + n]
// blockIdx.z selects a K-split: k in [z*kps, min(K,(z+1)*kps)), output at
// C + z*c_split.
template <int BM, int BN, int BK, int TM, int TN, bool TA, bool TB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
k_gemm(int M, int N, int K, const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb,
       float* __restrict__ C, int ldc, int64_t c_split, int kps, Epi ep) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int A_LD = (BM * BK) / NT;  // elements per thread per tile
  constexpr int B_LD = (BN * BK) / NT;
  static_assert(A_LD >= 1 && B_LD >= 1, "tile too small for the thread count");
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];

  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN);
  const int ty = tid / (BN / TN);
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int kz0 = blockIdx.z * kps;
  const int kz1 = min(K, kz0 + kps);
  C += (int64_t)blockIdx.z * c_split;

  float ra[A_LD], rb[B_LD];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int i = 0; i < A_LD; ++i) {
      const int idx = tid + i * NT;
      int m, k;
      if (TA) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      const int gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < M && gk < kz1) ? __ldg(TA ? A + (int64_t)gk * lda + gm : A + (int64_t)gm * lda + gk) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < B_LD; ++i) {
      const int idx = tid + i * NT;
      int n, k;
      if (TB) { n = idx / BK; k = idx % BK; } else { k = idx / BN; n = idx % BN; }
      const int gn = n0 + n, gk = k0 + k;
      rb[i] = (gn < N && gk < kz1) ? __ldg(TB ? B + (int64_t)gn * ldb + gk : B + (int64_t)gk * ldb + gn) : 0.f;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int i = 0; i < A_LD; ++i) {
      const int idx = tid + i * NT;
      int m, k;
      if (TA) { k = idx / BM; m = idx % BM; } else { m = idx / BK; k = idx % BK; }
      As[buf][k][m] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < B_LD; ++i) {
      const int idx = tid + i * NT;
      int n, k;
      if (TB) { n = idx / BK; k = idx % BK; } else { k = idx / BN; n = idx % BN; }
      Bs[buf][k][n] = rb[i];
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  int buf = 0;
  if (kz0 < kz1) {
    load_tile(kz0);
    store_tile(0);
  }
  __syncthreads();
  for (int k0 = kz0; k0 < kz1; k0 += BK) {
    const bool more = k0 + BK < kz1;
    if (more) load_tile(k0 + BK);  // global loads in flight during the FFMAs
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][k][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[buf][k][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_tile(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + tx * TN + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (ep.kind == EPI_BIAS_ACT) {
        v += ep.bias[gn];
        if (ep.lrelu) v = v > 0.f ? v : v * ep.alpha;
      } else if (ep.kind == EPI_ACT_GRAD) {
        v *= (ep.H[(int64_t)gm * ep.ldh + gn] > 0.f) ? 1.f : ep.alpha;
      }
      C[(int64_t)gm * ldc + gn] = v;
    }
  }
}

template <int BM, int BN, int BK, int TM, int TN>
static void gemm_cfg(bool ta, bool tb, dim3 grid, cudaStream_t st, int M, int N, int K, const float* A, int lda,
                     const float* B, int ldb, float* C, int ldc, int64_t c_split, int kps, const Epi& ep) {
  constexpr int NT = (BM / TM) * (BN / TN);
  if (!ta && !tb) k_gemm<BM, BN, BK, TM, TN, false, false><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  else if (!ta && tb) k_gemm<BM, BN, BK, TM, TN, false, true><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  else if (ta && !tb) k_gemm<BM, BN, BK, TM, TN, true, false><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  else k_gemm<BM, BN, BK, TM, TN, true, true><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  count_launch();
}

void launch_gemm(bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                 float* C, int ldc, const Epi& ep, int splits, int64_t c_split, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  if (splits < 1) splits = 1;
  int kps = (K + splits - 1) / splits;
  kps = ((kps + 7) / 8) * 8;
  auto blocks = [&](int bm, int bn) { return (int64_t)((M + bm - 1) / bm) * ((N + bn - 1) / bn) * splits; };
  if (M >= 128 && N >= 96 && blocks(128, 128) >= 2 * 148) {
    dim3 grid((M + 127) / 128, (N + 127) / 128, splits);
    gemm_cfg<128, 128, 8, 8, 8>(ta, tb, grid, st, M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  } else if (M >= 64 && N >= 48 && blocks(64, 64) >= 148) {
    dim3 grid((M + 63) / 64, (N + 63) / 64, splits);
    gemm_cfg<64, 64, 8, 4, 4>(ta, tb, grid, st, M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  } else if (N <= 8) {
    dim3 grid((M + 63) / 64, (N + 7) / 8, splits);
    gemm_cfg<64, 8, 8, 4, 2>(ta, tb, grid, st, M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  } else {
    dim3 grid((M + 31) / 32, (N + 31) / 32, splits);
    gemm_cfg<32, 32, 8, 2, 2>(ta, tb, grid, st, M, N, K, A, lda, B, ldb, C, ldc, c_split, kps, ep);
  }
}

// ---------------------------------------------------------------- column sums
// part[z][n] = sum over rows r in split z (ascending) of X[r][n].
__global__ void k_colsum(const float* __restrict__ X, int rows, int cols, int ldx, int rps,
                         float* __restrict__ part) {
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int z = blockIdx.y;
  const int r0 = z * rps, r1 = min(rows, r0 + rps);
  __shared__ float red[8][33];
  float acc = 0.f;
  if (n < cols)
    for (int r = r0 + threadIdx.y; r < r1; r += 8) acc += X[(int64_t)r * ldx + n];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && n < cols) {
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) v += red[i][threadIdx.x];
    part[(int64_t)z * cols + n] = v;
  }
}

void launch_colsum(const float* X, int rows, int cols, int ldx, int splits, float* part, cudaStream_t st) {
  const int rps = (rows + splits - 1) / splits;
  dim3 grid((cols + 31) / 32, splits);
  k_colsum<<<grid, dim3(32, 8), 0, st>>>(X, rows, cols, ldx, rps, part);
  count_launch();
}

// out[i] = (accumulate ? out[i] : 0) + scale * sum_{p ascending} part[p][i]
__global__ void k_reduce_parts(const float* __restrict__ part, int nparts, int64_t n, float* __restrict__ out,
                               float scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int p = 0; p < nparts; ++p) v += part[(int64_t)p * n + i];
    out[i] = v * scale;
  }
}

void launch_reduce_parts(const float* part, int nparts, int64_t n, float* out, float scale, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  k_reduce_parts<<<blocks, 256, 0, st>>>(part, nparts, n, out, scale);
  count_launch();
}

// ---------------------------------------------------------------- head
// Last discriminator layer (H -> 1) fused with the loss and its gradient.
// One warp per row at a time; lane j owns features j, j+32, ...
//   z = H[r] . w + b ; t = (r < n_real) ? 1 : label_rest
//   loss term = t softplus(-z) + (1 - t) softplus(z)     (accumulated in fp64)
//   dz = (sigmoid(z) - t) * scale
//   dZprev[r][j] = dz * w[j] * lrelu'(H[r][j])
//   part_w[block][j] += dz * H[r][j], part_b[block] += dz (fixed order)
template <int HD>
__global__ void __launch_bounds__(256) k_head(const float* __restrict__ Hm, int M, const float* __restrict__ w, const float* __restrict__ bptr,
                                              int n_real, float label_rest, float scale, float alpha,
                                              float* __restrict__ logits, float* __restrict__ dZprev,
                                              float* __restrict__ part, double* __restrict__ loss_part, int want_wgrad) {
  constexpr int PER = (HD + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int gw = blockIdx.x * nwarps + warp;
  const int total_w = gridDim.x * nwarps;
  float wv[PER], gwacc[PER];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int j = lane + 32 * p;
    wv[p] = (j < HD) ? w[j] : 0.f;
    gwacc[p] = 0.f;
  }
  const float b = *bptr;
  float gbacc = 0.f;
  double lacc = 0.0;
  for (int r = gw; r < M; r += total_w) {
    float h[PER];
    float dot = 0.f;
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int j = lane + 32 * p;
      h[p] = (j < HD) ? Hm[(int64_t)r * HD + j] : 0.f;
      dot = fmaf(h[p], wv[p], dot);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    const float z = dot + b;
    const float t = (r < n_real) ? 1.f : label_rest;
    const float dz = (sigmoid_f(z) - t) * scale;
    if (lane == 0) {
      logits[r] = z;
      lacc += (double)(t * softplus_neg(z) + (1.f - t) * softplus_neg(-z));
    }
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int j = lane + 32 * p;
      if (j < HD) {
        dZprev[(int64_t)r * HD + j] = dz * wv[p] * (h[p] > 0.f ? 1.f : alpha);
        gwacc[p] = fmaf(dz, h[p], gwacc[p]);
      }
    }
    gbacc += dz;
  }
  // fixed-order block reduction of the partials
  __shared__ float sw[8][HD + 1];
  __shared__ double sl[8];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int j = lane + 32 * p;
    if (j < HD) sw[warp][j] = gwacc[p];
  }
  if (lane == 0) { sw[warp][HD] = gbacc; sl[warp] = lacc; }
  __syncthreads();
  if (want_wgrad) {
    for (int j = threadIdx.x; j <= HD; j += blockDim.x) {
      float v = 0.f;
      for (int i = 0; i < nwarps; ++i) v += sw[i][j];
      part[(int64_t)blockIdx.x * (HD + 1) + j] = v;
    }
  }
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int i = 0; i < nwarps; ++i) v += sl[i];
    loss_part[blockIdx.x] = v;
  }
}

int head_blocks() { return 148 * 2; }

void launch_head(const float* H, int M, int hd, const float* w, const float* b, int n_real, float label_rest,
                 float scale, float alpha, float* logits, float* dZprev, float* part, double* loss_part,
                 bool want_wgrad, cudaStream_t st) {
  const int blocks = head_blocks();
  switch (hd) {
    case 64: k_head<64><<<blocks, 256, 0, st>>>(H, M, w, b, n_real, label_rest, scale, alpha, logits, dZprev, part, loss_part, want_wgrad); break;
    case 128: k_head<128><<<blocks, 256, 0, st>>>(H, M, w, b, n_real, label_rest, scale, alpha, logits, dZprev, part, loss_part, want_wgrad); break;
    case 32: k_head<32><<<blocks, 256, 0, st>>>(H, M, w, b, n_real, label_rest, scale, alpha, logits, dZprev, part, loss_part, want_wgrad); break;
    case 256: k_head<256><<<blocks, 256, 0, st>>>(H, M, w, b, n_real, label_rest, scale, alpha, logits, dZprev, part, loss_part, want_wgrad); break;
    default: break;  // validated at create time
  }
  count_launch();
}

// loss = scale * sum_{p ascending} loss_part[p] (finish_loss_block, common.cuh)
__global__ void __launch_bounds__(256) k_finish_loss(const double* __restrict__ loss_part, int nparts, double scale,
                                                     float* out, uint32_t* nonfinite) {
  __shared__ double sp[kLossCap];
  finish_loss_block(loss_part, nparts, scale, out, nonfinite, sp);
}

void launch_finish_loss(const double* loss_part, int nparts, double scale, float* out, uint32_t* nonfinite,
                        cudaStream_t st) {
  k_finish_loss<<<1, 256, 0, st>>>(loss_part, nparts, scale, out, nonfinite);
  count_launch();
}

}  // namespace sagips
