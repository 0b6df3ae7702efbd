// k_tc_layers.cu -- the discriminator MLP (paper preset: [2,128,128,128,128,1],
// P:297, R4) on the 5th-generation tensor cores, one kernel per layer pass,
// warp-specialised and persistent (one CTA per SM):
//
//   warps 0-3  producers: global fp32 rows -> bf16 (hi[, lo]) 128-byte-swizzled
//              shared-memory operand tiles (tc_util.cuh layout)
//   warps 4-7  epilogue : tcgen05.ld of the TMEM accumulator, fused math,
//              global stores (TMEM lane quarter = warp % 4)
//   warp  8    MMA      : one thread issues tcgen05.mma (kind::f16, fp32 acc)
//
// mbarrier pipeline: smem stage full/empty (producers <-> MMA), accumulator
// full/empty (MMA <-> epilogue), so staging of tile i+1, MMAs of tile i and
// the epilogue of tile i-1 overlap.
//
// k_tc_fwd<split, first, head>
//   first: the A tile is H1 = LeakyReLU(X W0^T + b0), recomputed from the
//          8-byte input rows instead of being stored (layer 0 never touches HBM)
//   head : the epilogue adds the last hidden layer's bias + LeakyReLU and the
//          head layer z = H.w + b, the BCE term, dz = (s(z) - t) * scale,
//          dZ = dz * w * LeakyReLU'(H), logits, and the head's weight-gradient
//          partials (warp-shuffle reduce-scatter, accumulated across tiles)
// k_tc_bwd<split, first, dy>
//   one pass over (dZ_l, H_{l-1}) computes both the dgrad dZ_{l-1} =
//   (dZ_l W_l) * LeakyReLU'(H_{l-1}) and the wgrad dW_l += dZ_l^T H_{l-1},
//   db_l += dZ_l^T 1 (persistent TMEM accumulators, one partial per CTA);
//   first: H1 recomputed from X; dy: the epilogue folds layer 0's input
//   gradient dy = dZ1 W0 (the G step needs dy, not dZ1).
// Precision: split = bf16x3 (hi*hi + hi*lo + lo*hi, fp32-class, PREC_FP32);
// !split = bf16 (PREC_BF16).
#include "ctx.h"
#include "tc_util.cuh"

namespace sagips {

using namespace tc;

namespace {

constexpr int kWarpsProd = 8;
constexpr int kWarpsEpi = 4;
constexpr int kThreads = 32 * (kWarpsProd + kWarpsEpi + 1);  // 416
constexpr int kProdThreads = 32 * kWarpsProd;
constexpr int kEpiWarp0 = kWarpsProd;                        // warps 8..11 (warp % 4 = TMEM lane quarter)
constexpr int kMmaWarp = kWarpsProd + kWarpsEpi;             // warp 12
constexpr uint32_t kTile = 128 * 128 * 2;                    // [128][128] bf16 SW128 tile
constexpr int kBatch = (128 * 16) / kProdThreads;            // chunk tasks per producer thread (8)

struct Params0 {  // layer-0 parameters for the on-the-fly H1, column-contiguous
  float w0x[128];
  float w0y[128];
  float b0[128];
};

__device__ __forceinline__ float lrelu(float z, float a) { return z > 0.f ? z : z * a; }

// write 8 values of row r, columns 8j..8j+7, into the SW128 planes (+ sign bits)
template <bool kSplit>
__device__ __forceinline__ void put_chunk(const float* x, int r, int j, uint8_t* hi, uint8_t* lo, uint8_t* mask) {
  const uint32_t off = sw128_chunk(r, j, 128);
  if (kSplit) {
    uint4 h, l;
    split_bf16(x, h, l);
    *reinterpret_cast<uint4*>(hi + off) = h;
    *reinterpret_cast<uint4*>(lo + off) = l;
  } else {
    *reinterpret_cast<uint4*>(hi + off) =
        make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
  }
  if (mask) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) m |= (x[i] > 0.f ? 1u : 0u) << i;
    mask[r * 16 + j] = (uint8_t)m;
  }
}

// stage rows [r0, r0+128) of a row-major [rows][128] fp32 matrix (zero rows
// beyond `rows`); all kBatch x 2 LDG.128 of a thread are issued before any is
// consumed (memory-level parallelism: 256 threads x 256 B in flight).
template <bool kSplit>
__device__ __forceinline__ void stage_from_global(const float* __restrict__ g, int64_t r0, int64_t rows, uint8_t* hi,
                                                  uint8_t* lo, uint8_t* mask, int t) {
  float4 buf[kBatch][2];
#pragma unroll
  for (int b = 0; b < kBatch; ++b) {
    const int q = t + b * kProdThreads;
    const int r = q >> 4, j = q & 15;
    const int64_t gr = r0 + r;
    if (gr < rows) {
      const float4* p = reinterpret_cast<const float4*>(g + gr * 128 + 8 * j);
      buf[b][0] = __ldg(p);
      buf[b][1] = __ldg(p + 1);
    } else {
      buf[b][0] = buf[b][1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
#pragma unroll
  for (int b = 0; b < kBatch; ++b) {
    const int q = t + b * kProdThreads;
    const float x[8] = {buf[b][0].x, buf[b][0].y, buf[b][0].z, buf[b][0].w,
                        buf[b][1].x, buf[b][1].y, buf[b][1].z, buf[b][1].w};
    put_chunk<kSplit>(x, q >> 4, q & 15, hi, lo, mask);
  }
}

// stage H1 = LeakyReLU(X W0^T + b0) for rows [r0, r0+128) of X [rows][2].
template <bool kSplit>
__device__ __forceinline__ void stage_h1(const float2* __restrict__ X, const Params0& p0, float alpha, int64_t r0,
                                         int64_t rows, uint8_t* hi, uint8_t* lo, uint8_t* mask, int t) {
  float2 xv[kBatch];
#pragma unroll
  for (int b = 0; b < kBatch; ++b) {
    const int q = t + b * kProdThreads;
    const int64_t gr = r0 + (q >> 4);
    xv[b] = gr < rows ? __ldg(X + gr) : make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int b = 0; b < kBatch; ++b) {
    const int q = t + b * kProdThreads;
    const int r = q >> 4, j = q & 15;
    float x[8];
    if (r0 + r < rows) {
      const float4 wa0 = *reinterpret_cast<const float4*>(&p0.w0x[8 * j]);
      const float4 wa1 = *reinterpret_cast<const float4*>(&p0.w0x[8 * j + 4]);
      const float4 wb0 = *reinterpret_cast<const float4*>(&p0.w0y[8 * j]);
      const float4 wb1 = *reinterpret_cast<const float4*>(&p0.w0y[8 * j + 4]);
      const float4 c0 = *reinterpret_cast<const float4*>(&p0.b0[8 * j]);
      const float4 c1 = *reinterpret_cast<const float4*>(&p0.b0[8 * j + 4]);
      const float wx[8] = {wa0.x, wa0.y, wa0.z, wa0.w, wa1.x, wa1.y, wa1.z, wa1.w};
      const float wy[8] = {wb0.x, wb0.y, wb0.z, wb0.w, wb1.x, wb1.y, wb1.z, wb1.w};
      const float bb[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = lrelu(fmaf(xv[b].x, wx[i], fmaf(xv[b].y, wy[i], bb[i])), alpha);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = 0.f;
    }
    put_chunk<kSplit>(x, r, j, hi, lo, mask);
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

}  // namespace

// ============================================================== forward
struct FwdArgs {
  const float* A;       // [rows][128] input activation (not first)
  const float* X;       // [rows][2] (first)
  const float* W0;      // [128][2] (first)
  const float* b0;      // [128] (first)
  const float* W;       // [128][128] this layer
  const float* bias;    // [128]
  float* C;             // [rows][128] output activation (not head)
  int64_t rows;
  float alpha;
  // head
  const float* w_head;  // [128]
  const float* b_head;  // [1]
  int64_t n_real;       // rows < n_real carry label 1, the rest label_rest
  float label_rest;
  float scale;          // 1/(number of rows in the mean)
  float* logits;        // [rows]
  float* dZ;            // [rows][128] gradient at the last hidden pre-activation
  float* part_head;     // [grid][129]: sum dz*H (128), sum dz
  double* loss_part;    // [grid]
  int want_wgrad;
};

template <bool kSplit, bool kFirst, bool kHead>
__global__ void __launch_bounds__(kThreads, 1) k_tc_fwd(FwdArgs a) {
  constexpr int P = kSplit ? 2 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = base;
  uint8_t* sA = base + P * kTile;  // 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + 2 * P * kTile);
  uint64_t* full = bars;        // [2]
  uint64_t* empty = bars + 2;   // [2]
  uint64_t* tfull = bars + 4;   // [2]
  uint64_t* tempty = bars + 6;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);  // [128]
  float* swh = sbias + 128;                                  // [128] head weights
  float* sred = swh + 128;                                   // [4][129] head partials
  double* sloss = reinterpret_cast<double*>(sred + 4 * 129 + 3);  // [4] (8-aligned below)
  sloss = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sloss) + 7) & ~uintptr_t(7));
  Params0* p0 = reinterpret_cast<Params0*>(sloss + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 32 * kWarpsProd);
      mbar_init(&empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kWarpsEpi);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<256>(tmem_slot);
  for (int i = tid; i < 128; i += kThreads) {
    sbias[i] = a.bias[i];
    if (kHead) swh[i] = a.w_head[i];
    if (kFirst) {
      p0->w0x[i] = a.W0[2 * i];
      p0->w0y[i] = a.W0[2 * i + 1];
      p0->b0[i] = a.b0[i];
    }
  }
  // the weight tile (B operand) is staged once by everyone
  for (int q = tid; q < 128 * 16; q += kThreads) {
    const int r = q >> 4, j = q & 15;
    const float4* p = reinterpret_cast<const float4*>(a.W + r * 128 + 8 * j);
    const float4 u = __ldg(p), v = __ldg(p + 1);
    const float x[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
    const uint32_t off = sw128_chunk(r, j, 128);
    if (kSplit) {
      uint4 h, l;
      split_bf16(x, h, l);
      *reinterpret_cast<uint4*>(sW + off) = h;
      *reinterpret_cast<uint4*>(sW + kTile + off) = l;
    } else {
      *reinterpret_cast<uint4*>(sW + off) =
          make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (warp < kWarpsProd) {
    // ---------------- producers
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
      const int s = i & 1;
      mbar_wait(&empty[s], ((i >> 1) & 1) ^ 1);
      uint8_t* st = sA + s * P * kTile;
      if (kFirst)
        stage_h1<kSplit>(reinterpret_cast<const float2*>(a.X), *p0, a.alpha, t * 128, a.rows, st, st + kTile, nullptr,
                         tid);
      else
        stage_from_global<kSplit>(a.A, t * 128, a.rows, st, st + kTile, nullptr, tid);
      fence_proxy_async_smem();
      mbar_arrive(&full[s]);
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
      const uint32_t bh = smem_u32(sW), bl = smem_u32(sW + kTile);
      for (int i = 0; i < nmine; ++i) {
        const int s = i & 1, b = i & 1;
        mbar_wait(&full[s], (i >> 1) & 1);
        mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(sA + s * P * kTile), al = ah + kTile;
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          const uint64_t adh = make_desc(ah + off, 16, 1024), bdh = make_desc(bh + off, 16, 1024);
          mma_bf16(d, adh, bdh, idesc, k > 0);
          if (kSplit) {
            mma_bf16(d, adh, make_desc(bl + off, 16, 1024), idesc, 1);
            mma_bf16(d, make_desc(al + off, 16, 1024), bdh, idesc, 1);
          }
        }
        mma_commit(&empty[s]);
        mma_commit(&tfull[b]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 4..7 -> TMEM lanes 32*(warp%4))
    const int q = warp & 3;
    const int lb = 32 * q;
    float gacc[4] = {0.f, 0.f, 0.f, 0.f};  // head: sum dz*H for columns 32c + lane
    float gbacc = 0.f;
    double lacc = 0.0;
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
      const int b = i & 1;
      mbar_wait(&tfull[b], (i >> 1) & 1);
      tc_fence_after();
      const int64_t row = t * 128 + lb + lane;
      const bool valid = row < a.rows;
      const uint32_t acc = tmem + (uint32_t)(b * 128) + ((uint32_t)lb << 16);
      if (!kHead) {
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
          if (valid) {
            float4* cp = reinterpret_cast<float4*>(a.C + row * 128 + 32 * c);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              cp[k] = make_float4(lrelu(v[4 * k] + sbias[32 * c + 4 * k], a.alpha),
                                  lrelu(v[4 * k + 1] + sbias[32 * c + 4 * k + 1], a.alpha),
                                  lrelu(v[4 * k + 2] + sbias[32 * c + 4 * k + 2], a.alpha),
                                  lrelu(v[4 * k + 3] + sbias[32 * c + 4 * k + 3], a.alpha));
          }
        }
      } else {
        // pass 1: z = H . w + b
        float dot = 0.f;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
#pragma unroll
          for (int k = 0; k < 32; ++k) dot = fmaf(lrelu(v[k] + sbias[32 * c + k], a.alpha), swh[32 * c + k], dot);
        }
        const float z = dot + *a.b_head;
        const float tl = (row < a.n_real) ? 1.f : a.label_rest;
        const float dz = valid ? (sigmoid_f(z) - tl) * a.scale : 0.f;
        if (valid) {
          a.logits[row] = z;
          lacc += (double)(tl * softplus_neg(z) + (1.f - tl) * softplus_neg(-z));
          gbacc += dz;
        }
        // pass 2: dZ = dz * w * LeakyReLU'(H) ; head weight gradient dz * H
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
          float g[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float zz = v[k] + sbias[32 * c + k];
            g[k] = dz * lrelu(zz, a.alpha);
            v[k] = dz * swh[32 * c + k] * (zz > 0.f ? 1.f : a.alpha);
          }
          if (valid) {
            float4* dp = reinterpret_cast<float4*>(a.dZ + row * 128 + 32 * c);
#pragma unroll
            for (int k = 0; k < 8; ++k) dp[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          }
          if (a.want_wgrad) {
            // reduce-scatter over the 32 rows of the warp: lane l ends with
            // the sum of column 32c + l
#pragma unroll
            for (int w = 16; w >= 1; w >>= 1) {
              const bool upper = (lane & w) != 0;
#pragma unroll
              for (int k = 0; k < w; ++k) {
                const float send = upper ? g[k] : g[k + w];
                const float recv = __shfl_xor_sync(0xffffffffu, send, w);
                g[k] = (upper ? g[k + w] : g[k]) + recv;
              }
            }
            gacc[c] += g[0];
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[b]);
    }
    if (kHead) {
      // per-CTA partials: loss (fp64), head weight gradient, head bias gradient
      for (int c = 0; c < 4; ++c) sred[q * 129 + 32 * c + lane] = gacc[c];
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
        gbacc += __shfl_xor_sync(0xffffffffu, gbacc, w);
        lacc += __shfl_xor_sync(0xffffffffu, lacc, w);
      }
      if (lane == 0) {
        sred[q * 129 + 128] = gbacc;
        sloss[q] = lacc;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kWarpsEpi));
      if (q == 0) {
        for (int j = lane; j <= 128; j += 32) {
          const float v = sred[j] + sred[129 + j] + sred[2 * 129 + j] + sred[3 * 129 + j];
          if (a.want_wgrad) a.part_head[(int64_t)blockIdx.x * 129 + j] = v;
        }
        if (lane == 0) a.loss_part[blockIdx.x] = sloss[0] + sloss[1] + sloss[2] + sloss[3];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// ============================================================== backward
struct BwdArgs {
  const float* dZ;     // [rows][128] gradient at layer l's pre-activation
  const float* H;      // [rows][128] H_{l-1} (not first)
  const float* X;      // [rows][2] (first)
  const float* W0;     // [128][2] (first)
  const float* b0;     // [128] (first)
  const float* W;      // [128][128] W_l
  int64_t rows;
  float alpha;
  float* dZout;        // [rows][128] dZ_{l-1} (store mode)
  float* dy;           // [rows][2] (dy mode)
  int want_wgrad;
  float* part;         // [grid][128][128]
  float* part_db;      // [grid][128]
};

template <bool kSplit, bool kFirst, bool kDy>
__global__ void __launch_bounds__(kThreads, 1) k_tc_bwd(BwdArgs a) {
  constexpr int P = kSplit ? 2 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = base;                     // W_l planes
  uint8_t* sZ = sW + P * kTile;           // dZ planes (one stage)
  uint8_t* sH = sZ + P * kTile;           // H planes (one stage)
  uint8_t* sOnes = sH + P * kTile;        // [16][128] ones, K-major SW128 (4 KB)
  uint8_t* sMask = sOnes + 4096;          // 2 x [128][16] sign bytes of H
  uint64_t* bars = reinterpret_cast<uint64_t*>(sMask + 2 * 2048);
  uint64_t* full = bars;                  // [1]
  uint64_t* empty = bars + 1;             // [1]
  uint64_t* tfull = bars + 2;             // [2]
  uint64_t* tempty = bars + 4;            // [2]
  uint64_t* wdone = bars + 6;             // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  float* sW0 = reinterpret_cast<float*>(tmem_slot + 4);  // [128][2] (dy mode)
  Params0* p0 = reinterpret_cast<Params0*>(sW0 + 256);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&full[0], 32 * kWarpsProd);
    mbar_init(&empty[0], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kWarpsEpi);
    }
    mbar_init(&wdone[0], 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  for (int i = tid; i < 128; i += kThreads) {
    if (kFirst) {
      p0->w0x[i] = a.W0[2 * i];
      p0->w0y[i] = a.W0[2 * i + 1];
      p0->b0[i] = a.b0[i];
    }
    if (kDy) {
      sW0[2 * i] = a.W0[2 * i];
      sW0[2 * i + 1] = a.W0[2 * i + 1];
    }
  }
  for (int i = tid; i < 4096 / 16; i += kThreads) {
    const uint32_t one2 = pack_bf16(1.f, 1.f);
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(one2, one2, one2, one2);
  }
  for (int q = tid; q < 128 * 16; q += kThreads) {
    const int r = q >> 4, j = q & 15;
    const float4* p = reinterpret_cast<const float4*>(a.W + r * 128 + 8 * j);
    const float4 u = __ldg(p), v = __ldg(p + 1);
    const float x[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
    const uint32_t off = sw128_chunk(r, j, 128);
    if (kSplit) {
      uint4 h, l;
      split_bf16(x, h, l);
      *reinterpret_cast<uint4*>(sW + off) = h;
      *reinterpret_cast<uint4*>(sW + kTile + off) = l;
    } else {
      *reinterpret_cast<uint4*>(sW + off) =
          make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc_w = tmem + 256, acc_b = tmem + 384;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (warp < kWarpsProd) {
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
      mbar_wait(&empty[0], (i & 1) ^ 1);             // MMAs of tile i-1 done with the stage
      mbar_wait(&tempty[i & 1], ((i >> 1) & 1) ^ 1);  // epilogue of tile i-2 done with mask[i&1]
      uint8_t* mask = sMask + (i & 1) * 2048;
      stage_from_global<kSplit>(a.dZ, t * 128, a.rows, sZ, sZ + kTile, nullptr, tid);
      if (kFirst)
        stage_h1<kSplit>(reinterpret_cast<const float2*>(a.X), *p0, a.alpha, t * 128, a.rows, sH, sH + kTile, mask,
                         tid);
      else
        stage_from_global<kSplit>(a.H, t * 128, a.rows, sH, sH + kTile, mask, tid);
      fence_proxy_async_smem();
      mbar_arrive(&full[0]);
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t id_d = make_idesc_bf16(128, 128, 0, 1);  // A = dZ (K-major), B = W (MN-major)
      constexpr uint32_t id_w = make_idesc_bf16(128, 128, 1, 1);  // A = dZ^T, B = H (both MN-major)
      constexpr uint32_t id_b = make_idesc_bf16(128, 16, 1, 0);   // A = dZ^T, B = ones (K-major)
      const uint32_t wh = smem_u32(sW), wl = wh + kTile;
      const uint32_t zh = smem_u32(sZ), zl = zh + kTile;
      const uint32_t hh = smem_u32(sH), hl = hh + kTile;
      const uint32_t on = smem_u32(sOnes);
      for (int i = 0; i < nmine; ++i) {
        const int b = i & 1;
        mbar_wait(&full[0], i & 1);
        mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32;  // K-major step (16 columns)
          const uint32_t km = k * 2048;                         // MN-major step (16 rows)
          // dgrad: D[rows][in] = dZ[rows][out] * W[out][in]
          const uint64_t zk_h = make_desc(zh + kk, 16, 1024);
          const uint64_t w_h = make_desc(wh + km, 16384, 1024);
          mma_bf16(d, zk_h, w_h, id_d, k > 0);
          if (kSplit) {
            mma_bf16(d, zk_h, make_desc(wl + km, 16384, 1024), id_d, 1);
            mma_bf16(d, make_desc(zl + kk, 16, 1024), w_h, id_d, 1);
          }
          if (a.want_wgrad) {
            const uint32_t acc0 = (i > 0 || k > 0) ? 1u : 0u;
            const uint64_t zm_h = make_desc(zh + km, 16384, 1024);
            const uint64_t h_h = make_desc(hh + km, 16384, 1024);
            const uint64_t od = make_desc(on + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024);
            mma_bf16(acc_w, zm_h, h_h, id_w, acc0);
            mma_bf16(acc_b, zm_h, od, id_b, acc0);
            if (kSplit) {
              const uint64_t zm_l = make_desc(zl + km, 16384, 1024);
              mma_bf16(acc_w, zm_h, make_desc(hl + km, 16384, 1024), id_w, 1);
              mma_bf16(acc_w, zm_l, h_h, id_w, 1);
              mma_bf16(acc_b, zm_l, od, id_b, 1);
            }
          }
        }
        mma_commit(&empty[0]);
        mma_commit(&tfull[b]);
      }
      mma_commit(&wdone[0]);
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int lb = 32 * q;
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
      const int b = i & 1;
      mbar_wait(&tfull[b], (i >> 1) & 1);
      tc_fence_after();
      const int r = lb + lane;
      const int64_t row = t * 128 + r;
      const bool valid = row < a.rows;
      const uint8_t* mask = sMask + b * 2048 + r * 16;
      const uint32_t acc = tmem + (uint32_t)(b * 128) + ((uint32_t)lb << 16);
      float dy0 = 0.f, dy1 = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(acc + 32 * c, v);
        const uint32_t mbits = *reinterpret_cast<const uint32_t*>(mask + 4 * c);
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] *= ((mbits >> k) & 1u) ? 1.f : a.alpha;
        if (kDy) {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            dy0 = fmaf(v[k], sW0[2 * (32 * c + k)], dy0);
            dy1 = fmaf(v[k], sW0[2 * (32 * c + k) + 1], dy1);
          }
        } else if (valid) {
          float4* dp = reinterpret_cast<float4*>(a.dZout + row * 128 + 32 * c);
#pragma unroll
          for (int k = 0; k < 8; ++k) dp[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        }
      }
      if (kDy && valid) reinterpret_cast<float2*>(a.dy)[row] = make_float2(dy0, dy1);
      tc_fence_before();
      mbar_arrive(&tempty[b]);
    }
    if (a.want_wgrad) {
      // TMEM lane = output feature o; 128 columns = input features
      const int o = lb + lane;
      float* dst = a.part + (int64_t)blockIdx.x * 128 * 128 + (int64_t)o * 128;
      if (nmine > 0) {
        mbar_wait(&wdone[0], 0);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld32(acc_w + 32 * c + ((uint32_t)lb << 16), v);
          float4* p = reinterpret_cast<float4*>(dst + 32 * c);
#pragma unroll
          for (int k = 0; k < 8; ++k) p[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        }
        float v[32];
        tmem_ld32(acc_b + ((uint32_t)lb << 16), v);
        a.part_db[(int64_t)blockIdx.x * 128 + o] = v[0];
      } else {
        for (int c = 0; c < 128; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        a.part_db[(int64_t)blockIdx.x * 128 + o] = 0.f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================== layer 0 grads
// dW0[c][0] = sum_r dZ1[r][c] x0_r, dW0[c][1] = sum_r dZ1[r][c] x1_r,
// db0[c] = sum_r dZ1[r][c]; per-block partials part[blk][c][3], fixed order.
__global__ void __launch_bounds__(256) k_l0_grads(const float* __restrict__ dZ1, const float2* __restrict__ X,
                                                  int64_t rows, int64_t rpb, float* __restrict__ part) {
  const int c = threadIdx.x & 127, half = threadIdx.x >> 7;
  const int64_t r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  float s0 = 0.f, s1 = 0.f, sb = 0.f;
  for (int64_t r = r0 + half; r < r1; r += 2) {
    const float g = dZ1[r * 128 + c];
    const float2 x = __ldg(X + r);
    s0 = fmaf(g, x.x, s0);
    s1 = fmaf(g, x.y, s1);
    sb += g;
  }
  __shared__ float red[2][128][3];
  red[half][c][0] = s0;
  red[half][c][1] = s1;
  red[half][c][2] = sb;
  __syncthreads();
  if (half == 0) {
    float* p = part + (int64_t)blockIdx.x * 384 + 3 * c;
    p[0] = red[0][c][0] + red[1][c][0];
    p[1] = red[0][c][1] + red[1][c][1];
    p[2] = red[0][c][2] + red[1][c][2];
  }
}

// out_w[c][0..1], out_b[c] from the partials
__global__ void k_l0_finish(const float* __restrict__ part, int nparts, float* __restrict__ dW0, float* __restrict__ db0) {
  const int c = threadIdx.x;
  if (c >= 128) return;
  float s0 = 0.f, s1 = 0.f, sb = 0.f;
  for (int p = 0; p < nparts; ++p) {
    s0 += part[(int64_t)p * 384 + 3 * c];
    s1 += part[(int64_t)p * 384 + 3 * c + 1];
    sb += part[(int64_t)p * 384 + 3 * c + 2];
  }
  dW0[2 * c] = s0;
  dW0[2 * c + 1] = s1;
  db0[c] = sb;
}

// head partials [grid][129] -> dW_head[128], db_head
__global__ void k_head_finish(const float* __restrict__ part, int nparts, float* __restrict__ dw, float* __restrict__ db) {
  const int j = threadIdx.x;
  if (j > 128) return;
  float s = 0.f;
  for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * 129 + j];
  if (j < 128) dw[j] = s;
  else *db = s;
}

// ============================================================== host
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = std::max(1, std::min(n, kMaxSms));
  }
  return n;
}

static size_t fwd_smem(bool split) {
  const int P = split ? 2 : 1;
  return 1024 + (size_t)3 * P * kTile + 8 * 8 + 16 + 4 * (128 + 128 + 4 * 129 + 4) + 8 * 4 + sizeof(Params0) + 64;
}
static size_t bwd_smem(bool split) {
  const int P = split ? 2 : 1;
  return 1024 + (size_t)3 * P * kTile + 4096 + 4096 + 8 * 8 + 16 + 4 * 256 + sizeof(Params0) + 64;
}

template <typename K>
static void allow_smem(K kern, size_t bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static void configure_layers() {
  static bool done = false;
  if (done) return;
  done = true;
#define SAGIPS_FWD(S, F, H) allow_smem(k_tc_fwd<S, F, H>, fwd_smem(S));
  SAGIPS_FWD(true, true, false) SAGIPS_FWD(true, false, false) SAGIPS_FWD(true, false, true)
  SAGIPS_FWD(false, true, false) SAGIPS_FWD(false, false, false) SAGIPS_FWD(false, false, true)
#undef SAGIPS_FWD
#define SAGIPS_BWD(S, F, D) allow_smem(k_tc_bwd<S, F, D>, bwd_smem(S));
  SAGIPS_BWD(true, false, false) SAGIPS_BWD(true, true, false) SAGIPS_BWD(true, true, true)
  SAGIPS_BWD(false, false, false) SAGIPS_BWD(false, true, false) SAGIPS_BWD(false, true, true)
#undef SAGIPS_BWD
}

int tc_layers_grid(int64_t rows) { return (int)std::min<int64_t>(std::max<int64_t>((rows + 127) / 128, 1), sm_count()); }

void launch_tc_fwd(bool split, int kind, const FwdLaunch& L, cudaStream_t st) {
  configure_layers();
  FwdArgs a{};
  a.A = L.A; a.X = L.X; a.W0 = L.W0; a.b0 = L.b0; a.W = L.W; a.bias = L.bias; a.C = L.C; a.rows = L.rows;
  a.alpha = L.alpha; a.w_head = L.w_head; a.b_head = L.b_head; a.n_real = L.n_real; a.label_rest = L.label_rest;
  a.scale = L.scale; a.logits = L.logits; a.dZ = L.dZ; a.part_head = L.part_head; a.loss_part = L.loss_part;
  a.want_wgrad = L.want_wgrad;
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = fwd_smem(split);
  if (split) {
    if (kind == 0) k_tc_fwd<true, true, false><<<grid, kThreads, sm, st>>>(a);
    else if (kind == 1) k_tc_fwd<true, false, false><<<grid, kThreads, sm, st>>>(a);
    else k_tc_fwd<true, false, true><<<grid, kThreads, sm, st>>>(a);
  } else {
    if (kind == 0) k_tc_fwd<false, true, false><<<grid, kThreads, sm, st>>>(a);
    else if (kind == 1) k_tc_fwd<false, false, false><<<grid, kThreads, sm, st>>>(a);
    else k_tc_fwd<false, false, true><<<grid, kThreads, sm, st>>>(a);
  }
  count_launch();
}

void launch_tc_bwd(bool split, bool first, bool dy, const BwdLaunch& L, cudaStream_t st) {
  configure_layers();
  BwdArgs a{};
  a.dZ = L.dZ; a.H = L.H; a.X = L.X; a.W0 = L.W0; a.b0 = L.b0; a.W = L.W; a.rows = L.rows; a.alpha = L.alpha;
  a.dZout = L.dZout; a.dy = L.dy; a.want_wgrad = L.want_wgrad; a.part = L.part; a.part_db = L.part_db;
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = bwd_smem(split);
  if (split) {
    if (!first) k_tc_bwd<true, false, false><<<grid, kThreads, sm, st>>>(a);
    else if (!dy) k_tc_bwd<true, true, false><<<grid, kThreads, sm, st>>>(a);
    else k_tc_bwd<true, true, true><<<grid, kThreads, sm, st>>>(a);
  } else {
    if (!first) k_tc_bwd<false, false, false><<<grid, kThreads, sm, st>>>(a);
    else if (!dy) k_tc_bwd<false, true, false><<<grid, kThreads, sm, st>>>(a);
    else k_tc_bwd<false, true, true><<<grid, kThreads, sm, st>>>(a);
  }
  count_launch();
}

int l0_grad_blocks() { return 296; }

void launch_l0_grads(const float* dZ1, const float* X, int64_t rows, float* part, float* dW0, float* db0,
                     cudaStream_t st) {
  const int nb = l0_grad_blocks();
  const int64_t rpb = (rows + nb - 1) / nb;
  k_l0_grads<<<nb, 256, 0, st>>>(dZ1, reinterpret_cast<const float2*>(X), rows, rpb, part);
  count_launch();
  k_l0_finish<<<1, 128, 0, st>>>(part, nb, dW0, db0);
  count_launch();
}

void launch_head_finish(const float* part, int nparts, float* dw, float* db, cudaStream_t st) {
  k_head_finish<<<1, 160, 0, st>>>(part, nparts, dw, db);
  count_launch();
}

}  // namespace sagips
