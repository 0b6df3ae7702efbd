// k_gen.cu -- the generator MLP (R4: [noise, H x depth, 6],
// LeakyReLU hidden layers, linear output) as three fused kernels: the
// generator is small (k = 1024 rows x ~51k parameters, ~0.3 GFLOP per step)
// and latency-bound, so each pass is one launch instead of a GEMM per layer.
//
//   k_gen_fwd   rows in blocks of kR per CTA through all layers (activations
//               in shared memory), every layer's output stored for the
//               backward, constrain (R1) fused on the output layer
//   k_gen_dgrad the same row blocks back through the layers:
//               dZ_{l-1} = (dZ_l W_l) * LeakyReLU'(H_{l-1})
//   k_gen_wgrad one CTA per 32 x 32 tile of every layer's weight gradient:
//               dW_l = dZ_l^T H_{l-1} over all rows (fixed order), plus
//               db_l = colsum(dZ_l); dW lands in the packet layout
// All sums run in a fixed order (deterministic); fp32 throughout.
#include "ctx.h"
#include "tc_util.cuh"

namespace sagips {
using tc::prefetch_l2;

namespace {
constexpr int kR = 8;         // rows per CTA (forward / dgrad)
constexpr int kGenMaxW = 128; // widest layer these kernels handle
constexpr int kGenThreads = 256;  // k_gen_wgrad: 16 x 16 output tiles
// the forward and the dgrad chain: 512 threads, thread (rb, o) of the 128 x 128
// fast path owns rows rb, rb + 4 (two rows: 16 warps per block hide the
// shared-memory latency better than 8 warps of four rows, ncu: 12.5% occupancy)
constexpr int kGenFT = 512;
constexpr int kRU = kR * kGenMaxW / kGenFT;  // rows per thread in the fast path
static_assert(kR == 8 && kRU == 2 && kGenFT == 4 * kGenMaxW, "the fast paths map 512 threads to 4 x 2 rows");
constexpr int kGenSplits = 8;  // wgrad: row splits (one partial each, reduced in a fixed order)
constexpr size_t kGenSmemMax = 227 * 1024;  // dynamic shared memory cap (all-layer weight staging)

__device__ __forceinline__ float lrelu_g(float z, float a) { return z > 0.f ? z : z * a; }
}  // namespace

struct GenArgs {
  int L;                          // linear layers
  int sizes[kMaxLayers + 1];
  int64_t w_off[kMaxLayers], b_off[kMaxLayers];
  const float* W;                 // all weights, layer l at w_off[l], [out][in] row-major
  const float* B;
  const float* noise;             // [k][sizes[0]]
  float* act[kMaxLayers];         // [k][sizes[l+1]] outputs of layer l (last: raw)
  float* dz[kMaxLayers];          // [k][sizes[l+1]] dLoss/dZ of layer l (last: draw, input)
  float* cbuf;                    // [k][6] constrained parameters
  float* dW;                      // packet layout (= W layout)
  float* dB;
  int k;
  float alpha;
  int tab;                        // constrain for the tabulated sampler (R32): c0 = sigmoid(raw0)
  // wgrad tiles: tile_base[l] = first blockIdx of layer l; tiles_i[l] = in-tiles per out-tile row
  int tile_base[kMaxLayers + 1];
  int tiles_i[kMaxLayers];
  // wgrad row splits (blockIdx.y): rows [y * split_rows, (y + 1) * split_rows);
  // with more than one, split y writes part + y * (wtot + btot) (dW then db, packet offsets)
  int split_rows;
  float* part;
  int64_t wtot, btot;
  // step prologue work riding on k_gen_fwd (the kernel before the sampler):
  // an L2 prefetch of the bootstrap shard (the sampler's random 8-byte
  // gathers then hit L2 instead of fetching 32-byte DRAM sectors) and the
  // zeroing of the step's histograms (no separate memset node)
  const char* prefetch;
  int64_t prefetch_bytes;
  uint32_t* zero_hist;
  int zero_words;
  // every layer's weights staged up front (cp.async, one group per layer in
  // use order) when they fit in shared memory: ws_off[l] = float offset of
  // layer l's copy after the row buffers; preload = 0 stages layer by layer
  // a1 inside the forward: the block draws its rows' noise (Philox + Box-
  // Muller, k_normals' arithmetic, stream NOISE of this step) and also stores
  // it to `noise`; gen_noise = 0 reads `noise`
  int gen_noise;
  float* noise_out;               // (gen_noise) where the drawn noise is stored: [k][sizes[0]]
  PhiloxKey noise_key;
  uint32_t noise_step, noise_rank;
  int preload;
  int ws_off[kMaxLayers];
  int ws_off_b[kMaxLayers];  // the dgrad's plain [out][in] copies (layers last .. 1)
};

// ---------------------------------------------------------------- async staging
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most n groups are pending (n is a small run-time count)
__device__ __forceinline__ void cp_async_wait(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
  }
}

// ---------------------------------------------------------------- forward
// Each layer's W is staged in shared memory, then each output accumulates its
// dot product in input order.  128 x 128 layers (the hidden ones): W staged
// with float4 loads all in flight (rows padded to 132 floats), thread (rb, o)
// computes output o of rows rb, rb + 2, rb + 4, rb + 6 from float4 reads of W
// and of the (broadcast) rows.  Other shapes: thread per (row, output), W rows
// padded to in + 1.
constexpr int kLdFast = kGenMaxW + 4;
__global__ void __launch_bounds__(kGenFT) k_gen_fwd(const __grid_constant__ GenArgs a) {
  extern __shared__ __align__(16) float gsm[];
  float(*buf)[kR][kGenMaxW] = reinterpret_cast<float(*)[kR][kGenMaxW]>(gsm);  // [2][kR][kGenMaxW]
  float* Ws = gsm + 2 * kR * kGenMaxW;                                         // [out][ld] (preload: base)
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * kR;
  const int in0 = a.sizes[0];
  if (a.prefetch && tid == 0) {  // this block's slice of the shard, in <= 32 KiB bulk prefetches
    const int64_t per = ((a.prefetch_bytes + gridDim.x - 1) / gridDim.x + 15) & ~(int64_t)15;
    const int64_t b0 = blockIdx.x * per, b1 = b0 + per < a.prefetch_bytes ? b0 + per : a.prefetch_bytes;
    for (int64_t o = b0; o < b1; o += 32768)
      prefetch_l2(a.prefetch + o, (uint32_t)(b1 - o < 32768 ? b1 - o : 32768));
  }
  if (a.zero_hist && blockIdx.x == 0)
    for (int i = tid; i < a.zero_words; i += kGenFT) a.zero_hist[i] = 0u;
  if (a.preload) {  // every layer's weights, layer order, one cp.async group each (same padded layouts)
    for (int l = 0; l < a.L; ++l) {
      const int in = a.sizes[l], out = a.sizes[l + 1];
      const float* W = a.W + a.w_off[l];
      float* dst = Ws + a.ws_off[l];
      if (in == kGenMaxW && out == kGenMaxW) {
        for (int idx = tid; idx < kGenMaxW * kGenMaxW / 4; idx += kGenFT)
          cp_async16(dst + (idx >> 5) * kLdFast + 4 * (idx & 31), W + 4 * idx);
      } else {
        for (int idx = tid; idx < out * in; idx += kGenFT) cp_async4(dst + (idx / in) * (in + 1) + idx % in, W + idx);
      }
      cp_async_commit();
    }
  }
  if (a.gen_noise) {  // the block's kR rows = values [r0 in0, (r0 + kR) in0): whole Philox calls (kR in0 % 4 == 0)
    for (int cl = tid; cl < kR * in0 / 4; cl += kGenFT) {
      const int64_t call = ((int64_t)r0 * in0) / 4 + cl;
      const uint4 w = philox_call(a.noise_key, (uint32_t)call, a.noise_step, a.noise_rank, kStreamNoise);
      float z[4];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const float ua = uniform_open01(p ? w.z : w.x);
        const float ub = uniform_open01(p ? w.w : w.y);
        const float rr = sqrtf(-2.0f * logf(ua));
        float sn, co;
        sincospif(2.0f * ub, &sn, &co);
        z[2 * p] = rr * co;
        z[2 * p + 1] = rr * sn;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int v = 4 * cl + q, r = v / in0, i = v % in0;
        const bool live = r0 + r < a.k;
        buf[0][r][i] = live ? z[q] : 0.f;
        if (live) a.noise_out[(int64_t)(r0 + r) * in0 + i] = z[q];
      }
    }
  } else {
    for (int idx = tid; idx < kR * in0; idx += kGenFT) {
      const int r = idx / in0, i = idx % in0;
      buf[0][r][i] = (r0 + r < a.k) ? a.noise[(int64_t)(r0 + r) * in0 + i] : 0.f;
    }
  }
  for (int l = 0; l < a.L; ++l) {
    const int in = a.sizes[l], out = a.sizes[l + 1];
    const bool fast = in == kGenMaxW && out == kGenMaxW;
    const int ld = fast ? kLdFast : in + 1;
    const float* W = a.W + a.w_off[l];
    const float* bias = a.B + a.b_off[l];
    if (a.preload) {
      cp_async_wait(a.L - 1 - l);  // this thread's copies of layers 0..l have landed
      __syncthreads();             // everyone's; and the previous layer is done with buf
      Ws = gsm + 2 * kR * kGenMaxW + a.ws_off[l];
    } else {
      __syncthreads();  // previous layer done with Ws / buf
    }
    if (a.preload) {
    } else if (fast) {
      constexpr int kV = kGenMaxW * kGenMaxW / 4 / kGenFT;
      float4 v[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(W) + tid + u * kGenFT);
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int idx = tid + u * kGenFT;  // float4 index: row idx / 32, columns 4 (idx % 32) ..
        *reinterpret_cast<float4*>(Ws + (idx >> 5) * kLdFast + 4 * (idx & 31)) = v[u];
      }
    } else {
      for (int idx = tid; idx < out * in; idx += kGenFT) Ws[(idx / in) * ld + idx % in] = __ldg(W + idx);
    }
    __syncthreads();
    const float(*src)[kGenMaxW] = buf[l & 1];
    float(*dst)[kGenMaxW] = buf[(l + 1) & 1];
    const bool hidden = l < a.L - 1;
    auto finish = [&](int r, int o, float acc) {
      acc += __ldg(bias + o);
      if (hidden) acc = lrelu_g(acc, a.alpha);
      dst[r][o] = acc;
      if (r0 + r < a.k) {
        a.act[l][(int64_t)(r0 + r) * out + o] = acc;
        if (!hidden) {  // a3: constrain (R1): c0 = raw, c1/c2 = softplus(raw)
          const int j = o % 3;
          a.cbuf[(int64_t)(r0 + r) * out + o] = (j == 0) ? (a.tab ? sigmoid_f(acc) : acc) : softplus_f(acc);
        }
      }
    };
    if (fast) {
      const int o = tid & (kGenMaxW - 1), rb = tid >> 7;
      const float* w = Ws + o * kLdFast;
      float acc[kRU] = {};
#pragma unroll 4
      for (int i = 0; i < kGenMaxW; i += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(w + i);
#pragma unroll
        for (int u = 0; u < kRU; ++u) {
          const float4 x = *reinterpret_cast<const float4*>(&src[rb + 4 * u][i]);
          acc[u] = fmaf(x.w, w4.w, fmaf(x.z, w4.z, fmaf(x.y, w4.y, fmaf(x.x, w4.x, acc[u]))));
        }
      }
#pragma unroll
      for (int u = 0; u < kRU; ++u) finish(rb + 4 * u, o, acc[u]);
    } else {
      for (int idx = tid; idx < kR * out; idx += kGenFT) {
        const int r = idx / out, o = idx % out;
        const float* w = Ws + o * ld;
        float acc = 0.f;
        for (int i = 0; i < in; ++i) acc = fmaf(src[r][i], w[i], acc);
        finish(r, o, acc);
      }
    }
  }
}

// ---------------------------------------------------------------- dgrad chain
// W_l staged in shared memory (lanes = consecutive inputs i read W[o][i]
// conflict-free), then each input accumulates over o in order; 128 x 128
// layers: thread (rb, i) does rows rb, rb + 2, rb + 4, rb + 6 with float4
// (broadcast) reads of the rows.
__global__ void __launch_bounds__(kGenFT) k_gen_dgrad(const __grid_constant__ GenArgs a) {
  extern __shared__ __align__(16) float gsm[];
  float(*buf)[kR][kGenMaxW] = reinterpret_cast<float(*)[kR][kGenMaxW]>(gsm);  // [2][kR][kGenMaxW]
  float* Ws = gsm + 2 * kR * kGenMaxW;                                         // [out][in]
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * kR;
  const int last = a.L - 1;
  const int outL = a.sizes[a.L];
  if (a.preload) {  // every layer's weights (use order: last .. 1), one cp.async group each, plain layout
    for (int l = last; l >= 1; --l) {
      const int in = a.sizes[l], out = a.sizes[l + 1];
      const float* W = a.W + a.w_off[l];
      float* dst = Ws + a.ws_off_b[l];
      if (in == kGenMaxW && out == kGenMaxW) {
        for (int idx = tid; idx < kGenMaxW * kGenMaxW / 4; idx += kGenFT) cp_async16(dst + 4 * idx, W + 4 * idx);
      } else {
        for (int idx = tid; idx < out * in; idx += kGenFT) cp_async4(dst + idx, W + idx);
      }
      cp_async_commit();
    }
  }
  for (int idx = tid; idx < kR * outL; idx += kGenFT) {
    const int r = idx / outL, o = idx % outL;
    buf[last & 1][r][o] = (r0 + r < a.k) ? a.dz[last][(int64_t)(r0 + r) * outL + o] : 0.f;
  }
  for (int l = last; l >= 1; --l) {
    const int in = a.sizes[l], out = a.sizes[l + 1];
    const bool fast = in == kGenMaxW && out == kGenMaxW;
    const float* W = a.W + a.w_off[l];
    if (a.preload) {
      cp_async_wait(l - 1);  // groups of layers last .. l have landed (l - 1 younger ones may be pending)
      __syncthreads();
      Ws = gsm + 2 * kR * kGenMaxW + a.ws_off_b[l];
    } else {
      __syncthreads();  // previous layer done with Ws / buf
    }
    if (a.preload) {
    } else if (fast) {
      constexpr int kV = kGenMaxW * kGenMaxW / 4 / kGenFT;
      float4 v[kV];
#pragma unroll
      for (int u = 0; u < kV; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(W) + tid + u * kGenFT);
#pragma unroll
      for (int u = 0; u < kV; ++u) reinterpret_cast<float4*>(Ws)[tid + u * kGenFT] = v[u];
    } else {
      for (int idx = tid; idx < out * in; idx += kGenFT) Ws[idx] = __ldg(W + idx);
    }
    __syncthreads();
    const float(*src)[kGenMaxW] = buf[l & 1];
    float(*dst)[kGenMaxW] = buf[(l - 1) & 1];
    auto finish = [&](int r, int i, float acc, float h) {
      acc *= (h > 0.f) ? 1.f : a.alpha;  // LeakyReLU'(Z) from the sign of H (R6)
      if (r0 + r >= a.k) acc = 0.f;
      dst[r][i] = acc;
      if (r0 + r < a.k) a.dz[l - 1][(int64_t)(r0 + r) * in + i] = acc;
    };
    if (fast) {
      const int i = tid & (kGenMaxW - 1), rb = tid >> 7;
      float h[kRU];
#pragma unroll
      for (int u = 0; u < kRU; ++u) {  // in flight during the sums
        const int r = rb + 4 * u;
        h[u] = (r0 + r < a.k) ? a.act[l - 1][(int64_t)(r0 + r) * in + i] : 0.f;
      }
      float acc[kRU] = {};
#pragma unroll 4
      for (int o = 0; o < kGenMaxW; o += 4) {
        const float w0 = Ws[o * kGenMaxW + i], w1 = Ws[(o + 1) * kGenMaxW + i];
        const float w2 = Ws[(o + 2) * kGenMaxW + i], w3 = Ws[(o + 3) * kGenMaxW + i];
#pragma unroll
        for (int u = 0; u < kRU; ++u) {
          const float4 x = *reinterpret_cast<const float4*>(&src[rb + 4 * u][o]);
          acc[u] = fmaf(x.w, w3, fmaf(x.z, w2, fmaf(x.y, w1, fmaf(x.x, w0, acc[u]))));
        }
      }
#pragma unroll
      for (int u = 0; u < kRU; ++u) finish(rb + 4 * u, i, acc[u], h[u]);
    } else {
      for (int idx = tid; idx < kR * in; idx += kGenFT) {
        const int r = idx / in, i = idx % in;
        float acc = 0.f;
        for (int o = 0; o < out; ++o) acc = fmaf(src[r][o], Ws[o * in + i], acc);
        const float h = (r0 + r < a.k) ? a.act[l - 1][(int64_t)(r0 + r) * in + i] : 0.f;
        finish(r, i, acc, h);
      }
    }
  }
}

// ---------------------------------------------------------------- wgrad
// blockIdx.x -> (layer l, out tile ob, in tile ib), blockIdx.y -> row split;
// thread (ty, tx) of 16 x 16 owns outputs (32ob + 2ty + {0,1}, 32ib + 2tx +
// {0,1}); the split's rows in chunks of 32, the next chunk's loads in flight
// (registers) while this one is summed.
__global__ void __launch_bounds__(kGenThreads) k_gen_wgrad(const __grid_constant__ GenArgs a) {
  __shared__ float sA[2][32][33];
  __shared__ float sB[2][32][33];
  int l = 0;
  while (l + 1 < a.L && (int)blockIdx.x >= a.tile_base[l + 1]) ++l;
  const int tb = blockIdx.x - a.tile_base[l];
  const int ob = tb / a.tiles_i[l], ib = tb % a.tiles_i[l];
  const int in = a.sizes[l], out = a.sizes[l + 1];
  const float* dZ = a.dz[l];
  const float* H = (l == 0) ? a.noise : a.act[l - 1];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  float dbacc = 0.f;
  float ra[4], rb[4];
  const int rs = blockIdx.y * a.split_rows, re = min(a.k, rs + a.split_rows);
  auto load = [&](int rc) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + u * kGenThreads;
      const int rr = idx >> 5, cc = idx & 31;
      const int r = rc + rr, o = 32 * ob + cc, i = 32 * ib + cc;
      ra[u] = (r < re && o < out) ? __ldg(dZ + (int64_t)r * out + o) : 0.f;
      rb[u] = (r < re && i < in) ? __ldg(H + (int64_t)r * in + i) : 0.f;
    }
  };
  auto stash = [&](int s) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = tid + u * kGenThreads;
      sA[s][idx >> 5][idx & 31] = ra[u];
      sB[s][idx >> 5][idx & 31] = rb[u];
    }
  };
  load(rs);
  stash(0);
  __syncthreads();
  int s = 0;
  for (int rc = rs; rc < re; rc += 32) {
    const bool more = rc + 32 < re;
    if (more) load(rc + 32);
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const float a0 = sA[s][rr][2 * ty], a1 = sA[s][rr][2 * ty + 1];
      const float b0 = sB[s][rr][2 * tx], b1 = sB[s][rr][2 * tx + 1];
      acc[0][0] = fmaf(a0, b0, acc[0][0]);
      acc[0][1] = fmaf(a0, b1, acc[0][1]);
      acc[1][0] = fmaf(a1, b0, acc[1][0]);
      acc[1][1] = fmaf(a1, b1, acc[1][1]);
    }
    if (ib == 0 && tid < 32) {
#pragma unroll 8
      for (int rr = 0; rr < 32; ++rr) dbacc += sA[s][rr][tid];
    }
    if (more) stash(s ^ 1);
    __syncthreads();
    s ^= 1;
  }
  const bool split = gridDim.y > 1;
  float* pbase = a.part + (int64_t)blockIdx.y * (a.wtot + a.btot);
  float* dW = (split ? pbase : a.dW) + a.w_off[l];
  float* dB = split ? pbase + a.wtot : a.dB;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int o = 32 * ob + 2 * ty + u, i = 32 * ib + 2 * tx + v;
      if (o < out && i < in) dW[(int64_t)o * in + i] = acc[u][v];
    }
  if (ib == 0 && tid < 32 && 32 * ob + tid < out) dB[a.b_off[l] + 32 * ob + tid] = dbacc;
}

// dW / db = sum over the row splits in split order
__global__ void __launch_bounds__(256) k_gen_wgrad_reduce(const float* __restrict__ part, int splits, int64_t wtot,
                                                          int64_t btot, float* __restrict__ dW, float* __restrict__ dB) {
  const int64_t n = wtot + btot;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int y = 0; y < splits; ++y) v += part[(int64_t)y * n + e];
    if (e < wtot) dW[e] = v;
    else dB[e - wtot] = v;
  }
}

// ---------------------------------------------------------------- host
bool gen_fused_ok(const sagips_ctx* c) {
  for (int l = 0; l <= c->G.L; ++l)
    if (c->G.sizes[l] > kGenMaxW) return false;
  return true;
}

static GenArgs gen_args(sagips_ctx* c) {
  GenArgs a{};
  const auto& G = c->G;
  a.L = G.L;
  for (int l = 0; l <= G.L; ++l) a.sizes[l] = G.sizes[l];
  int tb = 0;
  for (int l = 0; l < G.L; ++l) {
    a.w_off[l] = G.w_off[l];
    a.b_off[l] = G.b_off[l];
    a.act[l] = c->gAct[l];
    a.dz[l] = c->gdz_all[l];
    a.tile_base[l] = tb;
    a.tiles_i[l] = (G.sizes[l] + 31) / 32;
    tb += ((G.sizes[l + 1] + 31) / 32) * a.tiles_i[l];
  }
  a.tile_base[G.L] = tb;
  a.dz[G.L - 1] = c->draw;  // the output layer is linear: dZ_L = draw
  a.W = c->gW;
  a.B = c->gB;
  a.noise = c->noise;
  a.cbuf = c->cbuf;
  a.dW = c->g_dW;
  a.dB = c->g_dB;
  a.k = c->cfg.param_samples;
  a.alpha = c->cfg.leaky_slope;
  a.tab = c->cfg.sampler == SAGIPS_SAMPLER_TABULATED;
  a.wtot = G.nw;
  a.btot = G.nb;
  // row splits of 32-row multiples while the partials fit the scratch
  int splits = kGenSplits;
  while (splits > 1 && (int64_t)splits * (a.wtot + a.btot) > c->part_floats) splits >>= 1;
  a.split_rows = ((a.k + splits - 1) / splits + 31) / 32 * 32;
  a.part = c->part;
  // all layers' weights in shared memory at once when they fit (the forward's
  // padded layout; the dgrad's plain one is no larger)
  int off = 0;
  bool aligned = true;
  for (int l = 0; l < G.L; ++l) {
    const bool fast = G.sizes[l] == kGenMaxW && G.sizes[l + 1] == kGenMaxW;
    a.ws_off[l] = off;
    off += ((fast ? kGenMaxW * kLdFast : G.sizes[l + 1] * (G.sizes[l] + 1)) + 3) / 4 * 4;
    if (fast && (G.w_off[l] % 4) != 0) aligned = false;
  }
  a.preload = (aligned && G.L <= 8 && sizeof(float) * (2 * kR * kGenMaxW + off) <= kGenSmemMax) ? 1 : 0;
  int offb = 0;
  for (int l = G.L - 1; l >= 1; --l) {
    a.ws_off_b[l] = offb;
    offb += (G.sizes[l + 1] * G.sizes[l] + 3) / 4 * 4;
  }
  return a;
}

static size_t gen_smem(const GenArgs& a) {
  size_t w = (size_t)kGenMaxW * kLdFast;
  if (a.preload) {
    w = 0;
    for (int l = 0; l < a.L; ++l) {
      const bool fast = a.sizes[l] == kGenMaxW && a.sizes[l + 1] == kGenMaxW;
      w = (size_t)a.ws_off[l] + ((fast ? kGenMaxW * kLdFast : a.sizes[l + 1] * (a.sizes[l] + 1)) + 3) / 4 * 4;
    }
  }
  return sizeof(float) * (2 * kR * kGenMaxW + w);
}
static size_t gen_fwd_smem() { return kGenSmemMax; }  // the attribute: the largest launch

void launch_gen_fwd(sagips_ctx* c, cudaStream_t st, const void* prefetch, int64_t prefetch_bytes,
                    uint32_t* zero_hist, int zero_words, const uint32_t* noise_step) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gen_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gen_fwd_smem());
    configured = true;
  }
  GenArgs a = gen_args(c);
  a.prefetch = static_cast<const char*>(prefetch);
  a.prefetch_bytes = (prefetch_bytes / 16) * 16;
  a.zero_hist = zero_hist;
  a.zero_words = zero_words;
  if (noise_step && (kR * a.sizes[0]) % 4 == 0) {
    a.gen_noise = 1;
    a.noise_out = c->noise;
    a.noise_key = make_key(c->cfg.seed);
    a.noise_step = *noise_step;
    a.noise_rank = (uint32_t)c->cfg.rank;
  } else if (noise_step) {
    launch_normals(c->noise, (int64_t)c->cfg.param_samples * c->cfg.noise_dim, 1.0f, c->cfg.seed, *noise_step,
                   (uint32_t)c->cfg.rank, kStreamNoise, st);
  }
  k_gen_fwd<<<(a.k + kR - 1) / kR, kGenFT, gen_smem(a), st>>>(a);
  count_launch();
}

void launch_gen_predict(sagips_ctx* c, const float* noise, int k, float* c_out, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gen_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gen_fwd_smem());
    configured = true;
  }
  GenArgs a = gen_args(c);
  a.noise = noise;
  a.k = k;
  a.cbuf = c_out;
  k_gen_fwd<<<(a.k + kR - 1) / kR, kGenFT, gen_smem(a), st>>>(a);
  count_launch();
}

void launch_gen_bwd(sagips_ctx* c, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gen_dgrad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gen_fwd_smem());
    configured = true;
  }
  const GenArgs a = gen_args(c);
  k_gen_dgrad<<<(a.k + kR - 1) / kR, kGenFT, gen_smem(a), st>>>(a);
  count_launch();
  const int splits = (a.k + a.split_rows - 1) / a.split_rows;
  k_gen_wgrad<<<dim3(a.tile_base[a.L], splits), kGenThreads, 0, st>>>(a);
  count_launch();
  if (splits > 1) {
    const int64_t n = a.wtot + a.btot;
    k_gen_wgrad_reduce<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 4), 256, 0, st>>>(a.part, splits, a.wtot,
                                                                                          a.btot, a.dW, a.dB);
    count_launch();
  }
}

}  // namespace sagips
