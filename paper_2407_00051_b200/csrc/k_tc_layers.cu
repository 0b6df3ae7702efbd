// k_tc_layers.cu -- the discriminator MLP (paper preset: [2,128,128,128,128,1],
// P:297, R4) on the 5th-generation tensor cores, one kernel per layer pass,
// warp-specialised and persistent (one CTA per SM):
//
//   producer warps  global fp32 rows -> bf16 planes in 128-byte-swizzled
//                   shared-memory operand tiles (tc_util.cuh layout); each warp
//                   load instruction reads one contiguous 512-byte row; four
//                   register buffers keep three 4-row units of loads in
//                   flight; lane 0 of warp 0 bulk-prefetches the tiles two
//                   ahead into L2 (cp.async.bulk.prefetch.L2, no registers)
//   epilogue warps  tcgen05.ld of the TMEM accumulator (lane quarter = warp % 4;
//                   8 warps split the 128 columns in halves), fused math,
//                   stores transposed through a padded per-warp smem buffer so
//                   each store instruction writes whole lines
//   MMA warp        one thread issues tcgen05.mma (kind::f16, fp32 accumulate)
//
// mbarrier pipeline: smem stage full/free (producers <-> MMA), accumulator
// full/empty (MMA <-> epilogue).  SAGIPS_TRACE=1 records a per-tile timeline.
//
// k_tc_fwd<split, first, head>   (4 producer + 8 epilogue warps, 2 stages)
//   first: the A tile is H1 = LeakyReLU(X W0^T + b0), recomputed from the
//          8-byte input rows (layer 0 never touches HBM)
//   head : the epilogue adds the last hidden layer's bias + LeakyReLU and the
//          head layer z = H.w + b, the BCE term, dz = (s(z) - t) * scale,
//          dZ = dz * w * LeakyReLU'(H), the logits, and the head's weight-
//          gradient partials (warp-shuffle reduce-scatter across tiles)
// k_tc_bwd<split, first, dy>     (8 producer + 4 epilogue warps)
//   one pass over (dZ_l, H_{l-1}) computes the wgrad dW_l += dZ_l^T H_{l-1},
//   db_l += dZ_l^T 1 (persistent TMEM accumulators, one partial per CTA) and
//   then the dgrad dZ_{l-1} = (dZ_l W_l) * LeakyReLU'(H_{l-1}).  The H planes
//   are released as soon as the wgrad MMAs finish, so the producers write
//   H(i+1) while the dgrad of tile i runs.  Without wgrad (G step) only the
//   sign mask of H is staged.  first: H1 recomputed from X; dy: the epilogue
//   folds layer 0's input gradient dy = dZ1 W0 (the G step needs dy).
// Precision: split = bf16x4: x = hi + lo (two bf16), A*B = hi*hi + hi*lo +
// lo*hi + lo*lo (four MMAs; fp32-class), PREC_FP32;
// !split = bf16, PREC_BF16.
#include <cstdlib>

#include "ctx.h"
#include "tc_util.cuh"

namespace sagips {

using namespace tc;

namespace {

constexpr uint32_t kTile = 128 * 128 * 2;  // [128][128] bf16 SW128 tile
constexpr int kTStride = 36;               // 32-column transpose buffer row stride (floats)
constexpr uint32_t kTransWarp = 32 * kTStride * 4;
constexpr int kTStride16 = 20;             // 16-column transpose buffer row stride
constexpr uint32_t kTransWarp16 = 32 * kTStride16 * 4;

struct Params0 {  // layer-0 parameters for the on-the-fly H1, column-contiguous
  float w0x[128];
  float w0y[128];
  float b0[128];
};

__device__ __forceinline__ float lrelu(float z, float a) { return z > 0.f ? z : z * a; }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t x) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(x));
}
__device__ __forceinline__ void sts128f(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w));
}
__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

// named barrier among the epilogue warps
template <int EW>
__device__ __forceinline__ void epi_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
}

// ---- optional timeline trace (SAGIPS_TRACE=1): globaltimer stamps per tile
// for CTAs 0..3: 0 producer arrived full, 1 MMA started, 2 epilogue got the
// accumulator, 3 epilogue released it.
constexpr int kTraceLaunches = 32, kTraceCtas = 4, kTraceTiles = 256;
__device__ __forceinline__ void trace_pt(unsigned long long* tr, int i, int k) {
  if (tr && blockIdx.x < kTraceCtas && i < kTraceTiles) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[((size_t)blockIdx.x * kTraceTiles + i) * 4 + k] = t;
  }
}

// Shared-memory destinations of a staged tensor (0 = absent).
struct Dst {
  uint32_t hi, lo, mask;
};

// 4 values of row r, columns 4l..4l+3 -> the bf16 planes (8-byte halves of
// the 16-byte swizzle chunks) and/or 4 sign bits (> 0).
template <bool kSplit>
__device__ __forceinline__ void put4(float4 x, int r, int l, const Dst& d) {
  if (d.hi) {
    const uint32_t off = sw128_chunk(r, l >> 1, 128) + 8 * (l & 1);
    const __nv_bfloat162 h01 = __floats2bfloat162_rn(x.x, x.y), h23 = __floats2bfloat162_rn(x.z, x.w);
    sts64(d.hi + off, *reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
    if (kSplit) {
      const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
      const __nv_bfloat162 l01 = __floats2bfloat162_rn(x.x - f01.x, x.y - f01.y);
      const __nv_bfloat162 l23 = __floats2bfloat162_rn(x.z - f23.x, x.w - f23.y);
      sts64(d.lo + off, *reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
    }
  }
  if (d.mask)
    sts8(d.mask + r * 32 + l, (x.x > 0.f) | ((x.y > 0.f) << 1) | ((x.z > 0.f) << 2) | ((x.w > 0.f) << 3));
}

// ---- software-pipelined producers.  A "unit" is 4*PW consecutive rows of
// one staged tensor of one tile; lane l of producer warp w owns column
// float4 l of rows w, w+PW, w+2PW, w+3PW.  NB register buffers rotate: the
// loads of unit u+NB-1 are issued before unit u is converted.
constexpr int kRowsPerUnit = 8;  // rows per producer warp per unit
constexpr int kNB = 2;           // register buffers

struct Unit {
  const float* g;      // [rows][128] source (g == nullptr: H1 recomputed from X)
  const float2* X;
  int64_t r0;          // first global row of the unit
  int64_t rows;
  int trow;            // first tile row of the unit
};

template <int PW>
__device__ __forceinline__ void load_unit(float4 (&buf)[kRowsPerUnit], const Unit& u, int w, int l) {
#pragma unroll
  for (int i = 0; i < kRowsPerUnit; ++i) {
    const int64_t gr = u.r0 + w + PW * i;
    if (u.g) {
      buf[i] = gr < u.rows ? __ldg(reinterpret_cast<const float4*>(u.g + gr * 128) + l) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const float2 x = gr < u.rows ? __ldg(u.X + gr) : make_float2(0.f, 0.f);
      buf[i] = make_float4(x.x, x.y, gr < u.rows ? 1.f : 0.f, 0.f);
    }
  }
}

template <bool kSplit, int PW>
__device__ __forceinline__ void put_unit(const float4 (&buf)[kRowsPerUnit], const Unit& u, const Params0* p0,
                                         float alpha, const Dst& d, int w, int l) {
  float4 wx = make_float4(0.f, 0.f, 0.f, 0.f), wy = wx, bb = wx;
  if (!u.g) {
    wx = *reinterpret_cast<const float4*>(&p0->w0x[4 * l]);
    wy = *reinterpret_cast<const float4*>(&p0->w0y[4 * l]);
    bb = *reinterpret_cast<const float4*>(&p0->b0[4 * l]);
  }
#pragma unroll
  for (int i = 0; i < kRowsPerUnit; ++i) {
    const int r = u.trow + w + PW * i;
    float4 x = buf[i];
    if (!u.g) {  // H1 = LeakyReLU(X W0^T + b0); buf = (x0, x1, valid, 0)
      const float x0 = x.x, x1 = x.y;
      const bool ok = x.z != 0.f;
      x.x = ok ? lrelu(fmaf(x0, wx.x, fmaf(x1, wy.x, bb.x)), alpha) : 0.f;
      x.y = ok ? lrelu(fmaf(x0, wx.y, fmaf(x1, wy.y, bb.y)), alpha) : 0.f;
      x.z = ok ? lrelu(fmaf(x0, wx.z, fmaf(x1, wy.z, bb.z)), alpha) : 0.f;
      x.w = ok ? lrelu(fmaf(x0, wx.w, fmaf(x1, wy.w, bb.w)), alpha) : 0.f;
    }
    put4<kSplit>(x, r, l, d);
  }
}

// Drive `nunits` units through the kNB-buffer pipeline.
//   unit_of(u) -> Unit ; before_put(u) waits ; dest(u) -> Dst ; after_put(u) signals
template <bool kSplit, int PW, class UnitOf, class Before, class DestF, class After>
__device__ __forceinline__ void produce(int nunits, const Params0* p0, float alpha, int w, int l, UnitOf unit_of,
                                        Before before_put, DestF dest, After after_put) {
  float4 buf[kNB][kRowsPerUnit];
#pragma unroll
  for (int j = 0; j < kNB - 1; ++j)
    if (j < nunits) load_unit<PW>(buf[j], unit_of(j), w, l);
  for (int u = 0; u < nunits; u += kNB) {
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
      if (u + j < nunits) {
        if (u + j + kNB - 1 < nunits) load_unit<PW>(buf[(j + kNB - 1) % kNB], unit_of(u + j + kNB - 1), w, l);
        before_put(u + j);
        put_unit<kSplit, PW>(buf[j], unit_of(u + j), p0, alpha, dest(u + j), w, l);
        after_put(u + j);
      }
    }
  }
}

// W_l [128][128] fp32 -> planes (once per CTA, producer warps)
template <bool kSplit, int PW>
__device__ __forceinline__ void stage_weights(const float* __restrict__ W, uint32_t hi, uint32_t lo, int w, int l) {
  for (int t0 = 0; t0 < 128; t0 += kRowsPerUnit * PW) {
    float4 buf[kRowsPerUnit];
    const Unit u{W, nullptr, t0, 128, t0};
    load_unit<PW>(buf, u, w, l);
    put_unit<kSplit, PW>(buf, u, nullptr, 0.f, Dst{hi, lo, 0}, w, l);
  }
}

// bytes of tile t (rows [128t, 128t+128) clipped) of a [rows][cols] fp32 matrix
__device__ __forceinline__ uint32_t tile_bytes(int64_t t, int64_t rows, int cols) {
  const int64_t r0 = t * 128;
  if (r0 >= rows) return 0;
  return (uint32_t)(min((int64_t)128, rows - r0) * cols * 4);
}

// Epilogue store of a 32-row x 32-column chunk (tile rows lb..lb+31, columns
// c0..c0+31): lane = row holds v[32]; transpose through the warp's padded
// buffer (shared address sT) so 8 lanes write one contiguous 128-byte segment.
__device__ __forceinline__ void store_chunk(uint32_t sT, const float* v, float* __restrict__ gbase, int64_t tile_row0,
                                            int lb, int c0, int64_t rows, int lane) {
#pragma unroll
  for (int k = 0; k < 8; ++k) sts128f(sT + 4 * (lane * kTStride + 4 * k), v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int rr = it * 4 + (lane >> 3);
    const int cc = (lane & 7) * 4;
    const int64_t grow = tile_row0 + lb + rr;
    const float4 x = lds128f(sT + 4 * (rr * kTStride + cc));
    if (grow < rows) *reinterpret_cast<float4*>(gbase + grow * 128 + c0 + cc) = x;
  }
  __syncwarp();
}

// Same for 32 rows x 16 columns through a 32 x 20 buffer (the forward kernel's
// 8 epilogue warps cannot afford 4.5 KB each).
__device__ __forceinline__ void store_chunk16(uint32_t sT, const float* v, float* __restrict__ gbase, int64_t tile_row0,
                                              int lb, int c0, int64_t rows, int lane) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    sts128f(sT + 4 * (lane * kTStride16 + 4 * k), v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int rr = it * 8 + (lane >> 2);
    const int cc = (lane & 3) * 4;
    const int64_t grow = tile_row0 + lb + rr;
    const float4 x = lds128f(sT + 4 * (rr * kTStride16 + cc));
    if (grow < rows) *reinterpret_cast<float4*>(gbase + grow * 128 + c0 + cc) = x;
  }
  __syncwarp();
}

// MMA group for one K=16 step: D (+)= A*B with bf16 planes (split: 4 products)
template <bool kSplit>
__device__ __forceinline__ void mma_step(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl, uint32_t idesc,
                                         uint32_t acc) {
  mma_bf16(d, ah, bh, idesc, acc);
  if (kSplit) {
    mma_bf16(d, ah, bl, idesc, 1);
    mma_bf16(d, al, bh, idesc, 1);
    mma_bf16(d, al, bl, idesc, 1);
  }
}

}  // namespace

// ============================================================== forward
constexpr int kFwdPW = 4, kFwdEW = 8;
constexpr int kFwdThreads = 32 * (kFwdPW + kFwdEW + 1);  // 416
constexpr int kFwdMma = kFwdPW + kFwdEW;

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
  unsigned long long* trace;
};

template <bool kSplit, bool kFirst, bool kHead>
__global__ void __launch_bounds__(kFwdThreads, 1) k_tc_fwd(FwdArgs a) {
  constexpr int PW = kFwdPW, EW = kFwdEW;
  constexpr int P = kSplit ? 2 : 1;
  constexpr int kUnits = 128 / (kRowsPerUnit * PW);  // units per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = base;
  uint8_t* sA = base + P * kTile;  // 2 stages
  uint8_t* sTrans = sA + 2 * P * kTile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sTrans + EW * kTransWarp16);
  uint64_t* full = bars;        // [2]
  uint64_t* empty = bars + 2;   // [2]
  uint64_t* tfull = bars + 4;   // [2]
  uint64_t* tempty = bars + 6;  // [2]
  double* sloss = reinterpret_cast<double*>(bars + 8);     // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sloss + 4);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);  // [128]
  float* swh = sbias + 128;                                  // [128] head weights
  float* sred = swh + 128;                                   // [4][132] head partials
  float* pdot = sred + 4 * 132;                              // [2 parity][2 halves][128] partial dots
  Params0* p0 = reinterpret_cast<Params0*>(pdot + 512);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 32 * PW);
      mbar_init(&empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * EW);
    }
    fence_barrier_init();
  }
  if (warp == kFwdMma) tmem_alloc<256>(tmem_slot);
  for (int i = tid; i < 128; i += kFwdThreads) {
    sbias[i] = a.bias[i];
    if (kHead) swh[i] = a.w_head[i];
    if (kFirst) {
      p0->w0x[i] = a.W0[2 * i];
      p0->w0y[i] = a.W0[2 * i + 1];
      p0->b0[i] = a.b0[i];
    }
  }
  if (warp < PW) stage_weights<kSplit, PW>(a.W, smem_u32(sW), smem_u32(sW + kTile), warp, lane);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto tile_of = [&](int i) { return blockIdx.x + (int64_t)i * gridDim.x; };

  if (warp < PW) {
    // ---------------- producers
    const float2* X2 = reinterpret_cast<const float2*>(a.X);
    auto prefetch_tile = [&](int i) {
      if (i >= nmine) return;
      const int64_t t = tile_of(i);
      if (kFirst) prefetch_l2(X2 + t * 128, tile_bytes(t, a.rows, 2));
      else prefetch_l2(a.A + t * 128 * 128, tile_bytes(t, a.rows, 128));
    };
    if (warp == 0 && lane == 0) {
      prefetch_tile(1);
      prefetch_tile(2);
    }
    const uint32_t sA32 = smem_u32(sA);
    produce<kSplit, PW>(
        kUnits * nmine, p0, a.alpha, warp, lane,
        [&](int u) {
          const int64_t t = tile_of(u / kUnits);
          const int trow = (u % kUnits) * kRowsPerUnit * PW;
          return Unit{kFirst ? nullptr : a.A, X2, t * 128 + trow, a.rows, trow};
        },
        [&](int u) {
          if (u % kUnits == 0) {
            const int i = u / kUnits;
            if (warp == 0 && lane == 0 && i > 0) prefetch_tile(i + 2);
            mbar_wait(&empty[i & 1], ((i >> 1) & 1) ^ 1);
          }
        },
        [&](int u) {
          const uint32_t st = sA32 + ((u / kUnits) & 1) * P * kTile;
          return Dst{st, st + kTile, 0};
        },
        [&](int u) {
          if (u % kUnits == kUnits - 1) {
            fence_proxy_async_smem();
            mbar_arrive(&full[(u / kUnits) & 1]);
            if (warp == 0 && lane == 0) trace_pt(a.trace, u / kUnits, 0);
          }
        });
  } else if (warp == kFwdMma) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
      const uint32_t bh = smem_u32(sW), bl = smem_u32(sW + kTile);
      for (int i = 0; i < nmine; ++i) {
        const int s = i & 1, b = i & 1;
        mbar_wait(&full[s], (i >> 1) & 1);
        mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        trace_pt(a.trace, i, 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(sA + s * P * kTile), al = ah + kTile;
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          mma_step<kSplit>(d, make_desc(ah + off, 16, 1024), make_desc(al + off, 16, 1024),
                           make_desc(bh + off, 16, 1024), make_desc(bl + off, 16, 1024), idesc, k > 0);
        }
        mma_commit(&empty[s]);
        mma_commit(&tfull[b]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warp e -> TMEM lane quarter q, column half h
    const int e = warp - PW;
    const int q = warp & 3;
    const int h = e >> 2;
    const int lb = 32 * q;
    const int c_base = 64 * h;
    const uint32_t sT = smem_u32(sTrans) + e * kTransWarp16;
    float gacc[2] = {0.f, 0.f};  // head: sum dz*H for columns c_base + 32c + lane
    float gbacc = 0.f;
    double lacc = 0.0;
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = tile_of(i);
      const int b = i & 1;
      mbar_wait(&tfull[b], (i >> 1) & 1);
      if (e == 0 && lane == 0) trace_pt(a.trace, i, 2);
      tc_fence_after();
      const int64_t row = t * 128 + lb + lane;
      const bool valid = row < a.rows;
      const uint32_t acc = tmem + (uint32_t)(b * 128 + c_base) + ((uint32_t)lb << 16);
      if (!kHead) {
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = lrelu(v[k] + sbias[c_base + 32 * c + k], a.alpha);
          store_chunk16(sT, v, a.C, t * 128, lb, c_base + 32 * c, a.rows, lane);
          store_chunk16(sT, v + 16, a.C, t * 128, lb, c_base + 32 * c + 16, a.rows, lane);
        }
      } else {
        // pass 1: partial z = H . w over this warp's 64 columns
        float dot = 0.f;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int cc = c_base + 32 * c + k;
            dot = fmaf(lrelu(v[k] + sbias[cc], a.alpha), swh[cc], dot);
          }
        }
        float* pd = pdot + (i & 1) * 256;
        pd[h * 128 + lb + lane] = dot;
        epi_sync<EW>();
        const float z = pd[lb + lane] + pd[128 + lb + lane] + *a.b_head;
        const float tl = (row < a.n_real) ? 1.f : a.label_rest;
        const float dz = valid ? (sigmoid_f(z) - tl) * a.scale : 0.f;
        if (valid && h == 0) {
          a.logits[row] = z;
          lacc += (double)(tl * softplus_neg(z) + (1.f - tl) * softplus_neg(-z));
          gbacc += dz;
        }
        // pass 2: dZ = dz * w * LeakyReLU'(H) ; head weight gradient dz * H
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
          float g[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int cc = c_base + 32 * c + k;
            const float zz = v[k] + sbias[cc];
            g[k] = dz * lrelu(zz, a.alpha);
            v[k] = dz * swh[cc] * (zz > 0.f ? 1.f : a.alpha);
          }
          store_chunk16(sT, v, a.dZ, t * 128, lb, c_base + 32 * c, a.rows, lane);
          store_chunk16(sT, v + 16, a.dZ, t * 128, lb, c_base + 32 * c + 16, a.rows, lane);
          if (a.want_wgrad) {
            // reduce-scatter over the warp's 32 rows: lane l ends with column c_base + 32c + l
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
      if (e == 0 && lane == 0) trace_pt(a.trace, i, 3);
    }
    if (kHead) {
      // per-CTA partials: loss (fp64), head weight gradient, head bias gradient
      for (int c = 0; c < 2; ++c) sred[q * 132 + c_base + 32 * c + lane] = gacc[c];
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
        gbacc += __shfl_xor_sync(0xffffffffu, gbacc, w);
        lacc += __shfl_xor_sync(0xffffffffu, lacc, w);
      }
      if (lane == 0 && h == 0) {
        sred[q * 132 + 128] = gbacc;
        sloss[q] = lacc;
      }
      epi_sync<EW>();
      if (e == 0) {
        for (int j = lane; j <= 128; j += 32) {
          const float v = sred[j] + sred[132 + j] + sred[2 * 132 + j] + sred[3 * 132 + j];
          if (a.want_wgrad) a.part_head[(int64_t)blockIdx.x * 129 + j] = v;
        }
        if (lane == 0) a.loss_part[blockIdx.x] = sloss[0] + sloss[1] + sloss[2] + sloss[3];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kFwdMma) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// ============================================================== backward
constexpr int kBwdPW = 8, kBwdEW = 4;
constexpr int kBwdThreads = 32 * (kBwdPW + kBwdEW + 1);  // 416
constexpr int kBwdMma = kBwdPW + kBwdEW;

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
  unsigned long long* trace;
};

template <bool kSplit, bool kFirst, bool kDy>
__global__ void __launch_bounds__(kBwdThreads, 1) k_tc_bwd(BwdArgs a) {
  constexpr int PW = kBwdPW, EW = kBwdEW;
  constexpr int P = kSplit ? 2 : 1;
  constexpr int kUnitsT = 128 / (kRowsPerUnit * PW);  // units per tensor per tile
  constexpr int kUnits = 2 * kUnitsT;                 // H units first, then dZ units
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = base;                     // W_l planes
  uint8_t* sZ = sW + P * kTile;           // dZ planes (one stage)
  uint8_t* sH = sZ + P * kTile;           // H planes (one stage)
  uint8_t* sOnes = sH + P * kTile;        // [16][128] ones, K-major SW128 (4 KB)
  uint8_t* sMask = sOnes + 4096;          // 2 x [128][32] sign nibbles of H (8 KB)
  uint8_t* sTrans = sMask + 2 * 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sTrans + EW * kTransWarp);
  uint64_t* full_h = bars;                // [1] producers -> MMA: H planes (or mask) staged
  uint64_t* full_z = bars + 1;            // [1] producers -> MMA: dZ planes staged
  uint64_t* free_h = bars + 2;            // [1] MMA -> producers: wgrad done with H
  uint64_t* free_z = bars + 3;            // [1] MMA -> producers: all MMAs done with dZ
  uint64_t* tfull = bars + 4;             // [2]
  uint64_t* tempty = bars + 6;            // [2]
  uint64_t* wdone = bars + 8;             // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  float* sW0 = reinterpret_cast<float*>(tmem_slot + 4);  // [128][2] (dy mode)
  Params0* p0 = reinterpret_cast<Params0*>(sW0 + 256);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool wgrad = a.want_wgrad != 0;
  if (tid == 0) {
    mbar_init(&full_h[0], 32 * PW);
    mbar_init(&full_z[0], 32 * PW);
    mbar_init(&free_h[0], 1);
    mbar_init(&free_z[0], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * EW);
    }
    mbar_init(&wdone[0], 1);
    fence_barrier_init();
  }
  if (warp == kBwdMma) tmem_alloc<512>(tmem_slot);
  for (int i = tid; i < 128; i += kBwdThreads) {
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
  for (int i = tid; i < 4096 / 16; i += kBwdThreads) {
    const uint32_t one2 = pack_bf16(1.f, 1.f);
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(one2, one2, one2, one2);
  }
  if (warp < PW) stage_weights<kSplit, PW>(a.W, smem_u32(sW), smem_u32(sW + kTile), warp, lane);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc_w = tmem + 256, acc_b = tmem + 384;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto tile_of = [&](int i) { return blockIdx.x + (int64_t)i * gridDim.x; };

  if (warp < PW) {
    const float2* X2 = reinterpret_cast<const float2*>(a.X);
    auto prefetch_tile = [&](int i) {
      if (i >= nmine) return;
      const int64_t t = tile_of(i);
      prefetch_l2(a.dZ + t * 128 * 128, tile_bytes(t, a.rows, 128));
      if (kFirst) prefetch_l2(X2 + t * 128, tile_bytes(t, a.rows, 2));
      else prefetch_l2(a.H + t * 128 * 128, tile_bytes(t, a.rows, 128));
    };
    if (warp == 0 && lane == 0) {
      prefetch_tile(1);
      prefetch_tile(2);
    }
    const uint32_t zh = smem_u32(sZ), hh = smem_u32(sH), mk = smem_u32(sMask);
    produce<kSplit, PW>(
        kUnits * nmine, p0, a.alpha, warp, lane,
        [&](int u) {
          const int64_t t = tile_of(u / kUnits);
          const int k = u % kUnits;
          const bool isH = k < kUnitsT;
          const int trow = (k % kUnitsT) * kRowsPerUnit * PW;
          return Unit{isH ? (kFirst ? nullptr : a.H) : a.dZ, X2, t * 128 + trow, a.rows, trow};
        },
        [&](int u) {
          const int i = u / kUnits, k = u % kUnits;
          if (k == 0) {
            if (warp == 0 && lane == 0 && i > 0) prefetch_tile(i + 2);
            if (wgrad) mbar_wait(&free_h[0], (i & 1) ^ 1);   // wgrad of tile i-1 done with the H planes
            mbar_wait(&tempty[i & 1], ((i >> 1) & 1) ^ 1);   // epilogue of tile i-2 done with mask[i&1]
          } else if (k == kUnitsT) {
            mbar_wait(&free_z[0], (i & 1) ^ 1);              // all MMAs of tile i-1 done with dZ
          }
        },
        [&](int u) {
          const int i = u / kUnits, k = u % kUnits;
          if (k < kUnitsT) return Dst{wgrad ? hh : 0u, wgrad ? hh + kTile : 0u, mk + (i & 1) * 4096};
          return Dst{zh, zh + kTile, 0u};
        },
        [&](int u) {
          const int i = u / kUnits, k = u % kUnits;
          if (k == kUnitsT - 1) {
            fence_proxy_async_smem();
            mbar_arrive(&full_h[0]);
          } else if (k == kUnits - 1) {
            fence_proxy_async_smem();
            mbar_arrive(&full_z[0]);
            if (warp == 0 && lane == 0) trace_pt(a.trace, i, 0);
          }
        });
  } else if (warp == kBwdMma) {
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
        mbar_wait(&full_h[0], i & 1);
        mbar_wait(&full_z[0], i & 1);
        mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        trace_pt(a.trace, i, 1);
        tc_fence_after();
        if (wgrad) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t km = k * 2048;  // MN-major step (16 rows)
            const uint32_t acc0 = (i > 0 || k > 0) ? 1u : 0u;
            const uint64_t zm_h = make_desc(zh + km, 16384, 1024), zm_l = make_desc(zl + km, 16384, 1024);
            mma_step<kSplit>(acc_w, zm_h, zm_l, make_desc(hh + km, 16384, 1024), make_desc(hl + km, 16384, 1024),
                             id_w, acc0);
            const uint64_t od = make_desc(on + (k >> 2) * 2048 + (k & 3) * 32, 16, 1024);
            mma_bf16(acc_b, zm_h, od, id_b, acc0);
            if (kSplit) mma_bf16(acc_b, zm_l, od, id_b, 1);
          }
          mma_commit(&free_h[0]);
        }
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32;  // K-major step (16 columns)
          const uint32_t km = k * 2048;
          // dgrad: D[rows][in] = dZ[rows][out] * W[out][in]
          mma_step<kSplit>(d, make_desc(zh + kk, 16, 1024), make_desc(zl + kk, 16, 1024),
                           make_desc(wh + km, 16384, 1024), make_desc(wl + km, 16384, 1024), id_d, k > 0);
        }
        mma_commit(&free_z[0]);
        mma_commit(&tfull[b]);
      }
      mma_commit(&wdone[0]);
    }
    __syncwarp();
  } else {
    const int e = warp - PW;
    const int q = warp & 3;
    const int lb = 32 * q;
    const uint32_t sT = smem_u32(sTrans) + e * kTransWarp;
    const uint32_t mk = smem_u32(sMask);
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = tile_of(i);
      const int b = i & 1;
      mbar_wait(&tfull[b], (i >> 1) & 1);
      if (e == 0 && lane == 0) trace_pt(a.trace, i, 2);
      tc_fence_after();
      const int r = lb + lane;
      const int64_t row = t * 128 + r;
      const bool valid = row < a.rows;
      const uint32_t mask = mk + b * 4096 + r * 32;
      const uint32_t acc = tmem + (uint32_t)(b * 128) + ((uint32_t)lb << 16);
      float dy0 = 0.f, dy1 = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(acc + 32 * c, v);
        const uint2 mb = lds64(mask + 8 * c);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t word = k < 16 ? mb.x : mb.y;
          const uint32_t bit = ((k & 15) >> 2) * 8 + (k & 3);
          v[k] *= ((word >> bit) & 1u) ? 1.f : a.alpha;
        }
        if (kDy) {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            dy0 = fmaf(v[k], sW0[2 * (32 * c + k)], dy0);
            dy1 = fmaf(v[k], sW0[2 * (32 * c + k) + 1], dy1);
          }
        } else {
          store_chunk(sT, v, a.dZout, t * 128, lb, 32 * c, a.rows, lane);
        }
      }
      if (kDy && valid) reinterpret_cast<float2*>(a.dy)[row] = make_float2(dy0, dy1);
      tc_fence_before();
      mbar_arrive(&tempty[b]);
      if (e == 0 && lane == 0) trace_pt(a.trace, i, 3);
    }
    if (wgrad) {
      // TMEM lane = output feature o; 128 columns = input features
      const int o = lb + lane;
      float* dst = a.part + (int64_t)blockIdx.x * 128 * 128;
      if (nmine > 0) {
        mbar_wait(&wdone[0], 0);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld32(acc_w + 32 * c + ((uint32_t)lb << 16), v);
          store_chunk(sT, v, dst, 0, lb, 32 * c, 128, lane);
        }
        float v[32];
        tmem_ld32(acc_b + ((uint32_t)lb << 16), v);
        a.part_db[(int64_t)blockIdx.x * 128 + o] = v[0];
      } else {
        for (int c = 0; c < 128; c += 4) *reinterpret_cast<float4*>(dst + (int64_t)o * 128 + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        a.part_db[(int64_t)blockIdx.x * 128 + o] = 0.f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kBwdMma) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================== layer 0 grads
// dW0[c][0] = sum_r dZ1[r][c] x0_r, dW0[c][1] = sum_r dZ1[r][c] x1_r,
// db0[c] = sum_r dZ1[r][c]; per-block partials part[blk][c][3], fixed order.
// 32 rows per warp iteration, lane = 4 columns (float4): coalesced 512-B rows.
__global__ void __launch_bounds__(256) k_l0_grads(const float* __restrict__ dZ1, const float2* __restrict__ X,
                                                  int64_t rows, int64_t rpb, float* __restrict__ part) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0, sb = s0;
  for (int64_t r = r0 + w; r < r1; r += 8 * 4) {
    float4 g[4];
    float2 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t rr = r + 8 * u;
      g[u] = rr < r1 ? __ldg(reinterpret_cast<const float4*>(dZ1 + rr * 128) + l) : make_float4(0.f, 0.f, 0.f, 0.f);
      x[u] = rr < r1 ? __ldg(X + rr) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s0.x = fmaf(g[u].x, x[u].x, s0.x); s0.y = fmaf(g[u].y, x[u].x, s0.y);
      s0.z = fmaf(g[u].z, x[u].x, s0.z); s0.w = fmaf(g[u].w, x[u].x, s0.w);
      s1.x = fmaf(g[u].x, x[u].y, s1.x); s1.y = fmaf(g[u].y, x[u].y, s1.y);
      s1.z = fmaf(g[u].z, x[u].y, s1.z); s1.w = fmaf(g[u].w, x[u].y, s1.w);
      sb.x += g[u].x; sb.y += g[u].y; sb.z += g[u].z; sb.w += g[u].w;
    }
  }
  __shared__ float red[8][128][3];
  const float a0[4] = {s0.x, s0.y, s0.z, s0.w}, a1[4] = {s1.x, s1.y, s1.z, s1.w}, ab[4] = {sb.x, sb.y, sb.z, sb.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    red[w][4 * l + k][0] = a0[k];
    red[w][4 * l + k][1] = a1[k];
    red[w][4 * l + k][2] = ab[k];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 384; j += 256) {
    const int c = j / 3, e = j % 3;
    float v = 0.f;
    for (int i = 0; i < 8; ++i) v += red[i][c][e];
    part[(int64_t)blockIdx.x * 384 + j] = v;
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
  return 1024 + (size_t)3 * P * kTile + kFwdEW * kTransWarp16 + 8 * 8 + 8 * 4 + 16 +
         4 * (128 + 128 + 4 * 132 + 512) + sizeof(Params0) + 64;
}
static size_t bwd_smem(bool split) {
  const int P = split ? 2 : 1;
  return 1024 + (size_t)3 * P * kTile + 4096 + 8192 + kBwdEW * kTransWarp + 10 * 8 + 16 + 4 * 256 + sizeof(Params0) +
         64;
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

__device__ unsigned long long g_trace[kTraceLaunches][kTraceCtas * kTraceTiles * 4];
static int g_trace_on = -1;
static int g_trace_next = 0;
static unsigned long long* trace_slot() {
  if (g_trace_on < 0) {
    const char* e = getenv("SAGIPS_TRACE");
    g_trace_on = (e && e[0] == '1') ? 1 : 0;
  }
  if (!g_trace_on || g_trace_next >= kTraceLaunches) return nullptr;
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_trace);
  return reinterpret_cast<unsigned long long*>(p) + (size_t)(g_trace_next++) * kTraceCtas * kTraceTiles * 4;
}

size_t tc_trace_bytes() { return sizeof(unsigned long long) * kTraceLaunches * kTraceCtas * kTraceTiles * 4; }
int tc_trace_copy(void* host) {
  g_trace_next = 0;
  return cudaMemcpyFromSymbol(host, g_trace, tc_trace_bytes()) == cudaSuccess ? 0 : -1;
}

int tc_layers_grid(int64_t rows) { return (int)std::min<int64_t>(std::max<int64_t>((rows + 127) / 128, 1), sm_count()); }

void launch_tc_fwd(bool split, int kind, const FwdLaunch& L, cudaStream_t st) {
  configure_layers();
  FwdArgs a{};
  a.A = L.A; a.X = L.X; a.W0 = L.W0; a.b0 = L.b0; a.W = L.W; a.bias = L.bias; a.C = L.C; a.rows = L.rows;
  a.alpha = L.alpha; a.w_head = L.w_head; a.b_head = L.b_head; a.n_real = L.n_real; a.label_rest = L.label_rest;
  a.scale = L.scale; a.logits = L.logits; a.dZ = L.dZ; a.part_head = L.part_head; a.loss_part = L.loss_part;
  a.want_wgrad = L.want_wgrad;
  a.trace = trace_slot();
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = fwd_smem(split);
  if (split) {
    if (kind == FWD_FIRST) k_tc_fwd<true, true, false><<<grid, kFwdThreads, sm, st>>>(a);
    else if (kind == FWD_MID) k_tc_fwd<true, false, false><<<grid, kFwdThreads, sm, st>>>(a);
    else k_tc_fwd<true, false, true><<<grid, kFwdThreads, sm, st>>>(a);
  } else {
    if (kind == FWD_FIRST) k_tc_fwd<false, true, false><<<grid, kFwdThreads, sm, st>>>(a);
    else if (kind == FWD_MID) k_tc_fwd<false, false, false><<<grid, kFwdThreads, sm, st>>>(a);
    else k_tc_fwd<false, false, true><<<grid, kFwdThreads, sm, st>>>(a);
  }
  count_launch();
}

void launch_tc_bwd(bool split, bool first, bool dy, const BwdLaunch& L, cudaStream_t st) {
  configure_layers();
  BwdArgs a{};
  a.dZ = L.dZ; a.H = L.H; a.X = L.X; a.W0 = L.W0; a.b0 = L.b0; a.W = L.W; a.rows = L.rows; a.alpha = L.alpha;
  a.dZout = L.dZout; a.dy = L.dy; a.want_wgrad = L.want_wgrad; a.part = L.part; a.part_db = L.part_db;
  a.trace = trace_slot();
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = bwd_smem(split);
  if (split) {
    if (!first) k_tc_bwd<true, false, false><<<grid, kBwdThreads, sm, st>>>(a);
    else if (!dy) k_tc_bwd<true, true, false><<<grid, kBwdThreads, sm, st>>>(a);
    else k_tc_bwd<true, true, true><<<grid, kBwdThreads, sm, st>>>(a);
  } else {
    if (!first) k_tc_bwd<false, false, false><<<grid, kBwdThreads, sm, st>>>(a);
    else if (!dy) k_tc_bwd<false, true, false><<<grid, kBwdThreads, sm, st>>>(a);
    else k_tc_bwd<false, true, true><<<grid, kBwdThreads, sm, st>>>(a);
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
