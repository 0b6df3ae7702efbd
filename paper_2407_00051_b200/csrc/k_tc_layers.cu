// k_tc_layers.cu -- the discriminator MLP (paper preset [2,128,128,128,128,1],
// P:297, R4) on the 5th-generation tensor cores: one persistent,
// warp-specialised kernel per layer pass (one CTA per SM).
//
// Notation: linear layers W_0 [128x2], W_1..W_{L-2} [128x128],
// W_{L-1} [1x128] (head); Z_{l+1} = H_l W_l^T + b_l, H_l = LeakyReLU(Z_l),
// H_0 = X; G_l = dLoss/dZ_l.  dW_l = G_{l+1}^T H_l, db_l = colsum(G_{l+1}).
//
// Inter-kernel tensors live in HBM as "plane tiles": tile t (rows 128t ..
// 128t+127) is TB = P x 32 KiB at offset t*TB, plane 0 = bf16 hi(x), plane 1 =
// bf16 lo(x) = bf16(x - hi) (P = 2, fp32-class split; P = 1 for PREC_BF16);
// each plane is byte-identical to the SW128 shared-memory operand layout of
// tc_util.cuh, so a tile is moved by ONE 1-D bulk copy (TMA engine) with no
// register staging, and the same bytes serve as K-major (forward, dgrad) and
// MN-major (wgrad) operands.  The rows of a ragged last tile are zero.  Sign
// masks of the hidden activations (bit c of row r = H[r][c] > 0) are stored
// beside them (16 B per row) for the backward's LeakyReLU'.
//
// Warp roles (448 threads): warps 0-3 SIMT producers (first layer only: H_1
// is recomputed from the 8-byte input rows, it never touches HBM), warps 4-11
// epilogue (TMEM lane quarter = warp % 4, column half = (warp-4)/4), warp 12
// MMA issuer (one thread, tcgen05.mma kind::f16, fp32 accumulate in TMEM),
// warp 13 bulk loader (one thread).  Epilogues stage each 32-row x 64-column
// plane block (4 KiB, contiguous in HBM) in shared memory and store it with
// one bulk copy.
//
// Products (split): A*B ~= Ah*Bh + Ah*Bl + Al*Bh (bf16x3; the dropped Al*Bl is
// below the split's own representation error, tests/tools/precision_schemes.py).
//
// k_fwd<split, first, head>: Z = A W^T + b on 128-row tiles.
//   mid/first: H = LeakyReLU(Z) -> planes + mask.
//   head: H_{L-1} = LeakyReLU(Z), z = H.w + b, BCE term, logits,
//         dz = (sigmoid(z) - t) * scale, G = dz * w * LeakyReLU'(Z) -> planes;
//         head gradient partials (dz*H, dz).
// k_bwd<split, first, wgrad>: per tile, wgrad dW += G^T H and db += G^T 1
//   (persistent TMEM accumulators; the ones operand is a 512-byte
//   non-swizzled block) then dgrad G' = (G W) * LeakyReLU'(H) (the H stage is
//   released as soon as the wgrad MMAs finish).  Outputs: G' planes (mid), or,
//   for the first layer, the layer-0 gradients
//   dW_0 = G_1^T X, db_0 = colsum(G_1) (D step) or dy = G_1 W_0 (G step) in the
//   epilogue.  Without wgrad (G step) the H stage becomes a second G stage.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "ctx.h"
#include "tc_util.cuh"

namespace sagips {

using namespace tc;

namespace {

constexpr uint32_t kPlane = 128 * 128 * 2;   // one bf16 plane of a 128x128 tile
constexpr uint32_t kStg = 4096;              // per-epilogue-warp staging (32 rows x 128 B)
constexpr int kPW = 4, kEW = 8;
constexpr int kMmaWarp = kPW + kEW;          // 12
constexpr int kLoadWarp = kMmaWarp + 1;      // 13
constexpr int kThreads = 32 * (kLoadWarp + 1);  // 448
constexpr int kSmemLimit = 232448;           // 227 KiB opt-in per CTA
// first forward layer: plane FIFO + double-buffered staging (as the middle
// layers) instead of two whole-tile stages
constexpr bool kFirstFifo = false;  // measured slower (0.48 vs 0.43 ms, D step): producers wait on two plane slots

struct Params0 {  // layer-0 parameters, column-contiguous
  float w0x[128];
  float w0y[128];
  float b0[128];
};


__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}

// named barrier among the 8 epilogue warps
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEW) : "memory"); }

// ---- packed fp32 pairs: FADD2 / FMUL2 / FFMA2 (sm_100a), each lane rounded
// exactly as the scalar instruction (RN), one issue slot per pair
__device__ __forceinline__ uint64_t pk2(float2 a) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk2(uint64_t r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
// a * b + c, fused (as fmaf)
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return upk2(d);
}

// bf16x2 word {low half: bf16(a), high half: bf16(b)}, round to nearest even
__device__ __forceinline__ uint32_t bf16x2_rn(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
// hi = bf16(a,b), lo = bf16(a - hi, b - hi)
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  hi = bf16x2_rn(a, b);
  const float2 hf = make_float2(__uint_as_float(hi << 16), __uint_as_float(hi & 0xffff0000u));
  const float2 d = sub2(make_float2(a, b), hf);
  lo = bf16x2_rn(d.x, d.y);
}
// h = LeakyReLU(z) of a pair, split into hi / lo words.  LeakyReLU is
// max(z, a z): for 0 <= a < 1 (validated, R6) it equals (z > 0 ? z : a z) bit
// for bit (also for -0 and NaN) in two instructions.
__device__ __forceinline__ void lrelu_split2(float2 z, float2 alpha2, uint32_t& hi, uint32_t& lo) {
  const float2 t = mul2(z, alpha2);
  split2(fmaxf(z.x, t.x), fmaxf(z.y, t.y), hi, lo);
}
// Activation sign masks (16 B per row, 32 bits per 32-column block): in each
// block, column 2k is bit k and column 2k+1 is bit 16 + k, set iff
// bf16(H) > 0, from the packed hi word of the pair in one compare.  This is
// [Z > 0] except for 0 < Z < 2^-134 (bf16(H) underflows to +0), far below the
// GEMM's own rounding (R30).
__device__ __forceinline__ uint32_t pos_bits(uint32_t hi, int k) {
  uint32_t gt;
  asm("set.gt.u32.bf16x2 %0, %1, %2;" : "=r"(gt) : "r"(hi), "r"(0u));
  return gt & (0x00010001u << k);
}
// bit of column k (0..31) of a 32-column block in that layout
__host__ __device__ constexpr int mask_bit(int k) { return (k >> 1) + 16 * (k & 1); }

// 16 packed words = columns 32c..32c+31 of the warp's 64-column region, row
// `lane` of the warp's 32-row block -> the staging buffer (SW128 layout of
// rows 0..31 of one region: row r at r*128, chunk j at (j ^ (r % 8)) * 16).
__device__ __forceinline__ void stage_words(uint32_t stg, int lane, int c, const uint32_t* w) {
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const int j = 4 * c + jj;
    sts128(stg + lane * 128 + ((j ^ (lane & 7)) << 4), w[4 * jj], w[4 * jj + 1], w[4 * jj + 2], w[4 * jj + 3]);
  }
}

// staged block -> HBM (one 4 KiB bulk copy); called by the whole warp
__device__ __forceinline__ void flush_stage(uint32_t stg, uint8_t* dst, int lane) {
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    bulk_s2g(dst, stg, kStg);
    bulk_commit();
  }
}
// wait until the warp's previous bulk store has read the staging buffer
__device__ __forceinline__ void stage_free(int lane) {
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
}
// double-buffered staging: the buffer about to be written was used by the
// warp's second-to-last bulk store (the last one may still be reading)
__device__ __forceinline__ void stage_free_dbl(int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
}

// reduce-scatter over the warp's 32 rows: on return lane l holds the sum over
// lanes of g[l] (fixed order; g is destroyed)
__device__ __forceinline__ float colsum32(float (&g)[32], int lane) {
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
  return g[0];
}

// MMA group for one K = 16 step: D (+)= A*B (split: bf16x3)
template <bool kSplit>
__device__ __forceinline__ void mma_step(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl, uint32_t idesc,
                                         uint32_t acc) {
  mma_bf16(d, ah, bh, idesc, acc);
  if (kSplit) {
    mma_bf16(d, ah, bl, idesc, 1);
    mma_bf16(d, al, bh, idesc, 1);
  }
}

template <bool kSplit>
__device__ __forceinline__ void mma_step_warp(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                              uint32_t idesc, uint32_t acc) {
  mma_bf16_warp(d, ah, bh, idesc, acc);
  if (kSplit) {
    mma_bf16_warp(d, ah, bl, idesc, 1);
    mma_bf16_warp(d, al, bh, idesc, 1);
  }
}

// W [128][128] fp32 -> hi/lo planes (once per CTA; warps 0-3)
template <bool kSplit>
__device__ __forceinline__ void stage_weights(const float* __restrict__ W, uint32_t hi, uint32_t lo, int w, int l) {
#pragma unroll 1
  for (int r0 = w; r0 < 128; r0 += 8 * kPW) {
    float4 x[8];  // 8 independent loads in flight
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(W + (r0 + kPW * u) * 128) + l);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t off = sw128_chunk(r0 + kPW * u, l >> 1, 128) + 8 * (l & 1);
      uint32_t h0, h1, l0, l1;
      split2(x[u].x, x[u].y, h0, l0);
      split2(x[u].z, x[u].w, h1, l1);
      sts64(hi + off, h0, h1);
      if (kSplit) sts64(lo + off, l0, l1);
    }
  }
}

// SIMT producer of H_1 planes: rows row0 .. row0 + kRows - 1 of one tile
// (row0 % 8 == 0); lane l: channels 8(l % 16) .. 8(l % 16) + 7 (one 16-byte
// chunk) of the rows of parity l / 16, two rows per warp instruction; xr =
// lane i's prefetched input row row0 + i (i < kRows).  Z_1 = fma(x0, w0x,
// fma(x1, w0y, b0)) per channel, the order the backward recomputes it in.
// Rows past the end (ragged last tile) are written as zeros.
// Layer-0 parameters of lane l's channels 8(l % 16) .. + 7 as pairs, from the
// shared-memory copy or from global memory (W_0 [128][2], b_0 [128])
struct W0Lane {
  float2 wx[4], wy[4], bb[4];
};
__device__ __forceinline__ W0Lane w0_lane(const Params0* p0, int l) {
  const int jc = l & 15;
  W0Lane w;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    w.wx[p] = *reinterpret_cast<const float2*>(&p0->w0x[8 * jc + 2 * p]);
    w.wy[p] = *reinterpret_cast<const float2*>(&p0->w0y[8 * jc + 2 * p]);
    w.bb[p] = *reinterpret_cast<const float2*>(&p0->b0[8 * jc + 2 * p]);
  }
  return w;
}
__device__ __forceinline__ W0Lane w0_lane(const float* __restrict__ W0, const float* __restrict__ b0, int l) {
  const int jc = l & 15;
  W0Lane w;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(W0 + 2 * (8 * jc + 2 * p)));  // (x, y) of 2 channels
    w.wx[p] = make_float2(q.x, q.z);
    w.wy[p] = make_float2(q.y, q.w);
    w.bb[p] = __ldg(reinterpret_cast<const float2*>(b0 + 8 * jc + 2 * p));
  }
  return w;
}

template <bool kSplit, int kRows>
__device__ __forceinline__ void produce_h1(float2 xr, bool xvalid, const W0Lane& w, float alpha, uint32_t hi,
                                           uint32_t lo, int row0, int l) {
  static_assert(kRows % 8 == 0 && kRows <= 32, "rows");
  const int jc = l & 15, par = l >> 4;
  const float2 *wx = w.wx, *wy = w.wy, *bb = w.bb;
  const float2 alpha2 = make_float2(alpha, alpha);
  constexpr unsigned kNeed = kRows == 32 ? 0xffffffffu : ((1u << kRows) - 1u);
  const unsigned vbits = __ballot_sync(0xffffffffu, xvalid) & kNeed;
  // SW128 offset of (row row0 + 8 b + 2 u + par, chunk jc) = base + 1024 b + sw[u]
  const uint32_t base = (uint32_t)(jc >> 3) * 16384u + (uint32_t)(row0 >> 3) * 1024u;
  const int jp = (jc & 7) ^ par;
  uint32_t sw[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) sw[u] = (uint32_t)(2 * u + par) * 128u + ((uint32_t)(jp ^ (2 * u)) << 4);
  auto rows = [&](auto ragged) {
#pragma unroll
    for (int it = 0; it < kRows / 2; ++it) {
      const int src = 2 * it + par;
      const float x0 = __shfl_sync(0xffffffffu, xr.x, src), x1 = __shfl_sync(0xffffffffu, xr.y, src);
      const float2 X0 = make_float2(x0, x0), X1 = make_float2(x1, x1);
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 z = fma2(X0, wx[p], fma2(X1, wy[p], bb[p]));
        if constexpr (decltype(ragged)::value) {
          const float ok = ((vbits >> src) & 1u) ? 1.f : 0.f;
          const float2 t = mul2(z, alpha2);
          split2(ok * fmaxf(z.x, t.x), ok * fmaxf(z.y, t.y), hw[p], lw[p]);
        } else {
          lrelu_split2(z, alpha2, hw[p], lw[p]);
        }
      }
      const uint32_t off = base + (uint32_t)(it >> 2) * 1024u + sw[it & 3];
      sts128(hi + off, hw[0], hw[1], hw[2], hw[3]);
      if (kSplit) sts128(lo + off, lw[0], lw[1], lw[2], lw[3]);
    }
  };
  if (vbits == kNeed)
    rows(std::false_type{});
  else
    rows(std::true_type{});
}

// ---- optional timeline trace (SAGIPS_TRACE=1): globaltimer stamps per tile
// for CTAs 0..3: 0 operands staged, 1 MMA started, 2 epilogue got the
// accumulator, 3 epilogue released it.
constexpr int kTraceLaunches = 32, kTraceCtas = 4, kTraceTiles = 256;
__device__ __forceinline__ void trace_pt(unsigned long long* tr, int j, int i, int k) {
  if (tr && j < kTraceCtas && i < kTraceTiles) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[((size_t)j * kTraceTiles + i) * 4 + k] = t;
  }
}

__device__ __forceinline__ void check_smem_alignment(const void* p) {
  if (smem_u32(p) & 1023u) __trap();  // SW128 operands need 1024-byte alignment
}

// ---- inter-CTA dataflow (ring buffers with per-tile counters; unused by the
// per-layer kernels, whose tensors are whole, rdy / done == nullptr): plane tiles pass
// between layer roles through ring buffers in global memory (L2-resident);
// per-tile counters carry release/acquire ordering.
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// relaxed poll (an acquire load invalidates the SM's L1 on every poll)
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// spin (relaxed) until *p >= target, then one acquire load; a dataflow stall
// of > 4 s is a bug -> trap (no hang)
__device__ __noinline__ void wait_flag(const uint32_t* p, uint32_t target) {
  if (ld_relaxed(p) < target) {
    const unsigned long long t0 = globaltimer();
    while (ld_relaxed(p) < target) {
      __nanosleep(64);
      if (globaltimer() - t0 > 4000000000ull) __trap();
    }
  }
  (void)ld_acquire(p);
}
// ---- wait accounting (SAGIPS_TRACE=1, pipelined step): ns per CTA spent in
// 0 loader: upstream tile ready  1 loader: stage free  2 MMA: operands  3 MMA:
// accumulator free  4 epilogue: output slot free  5 epilogue: accumulator  6
// epilogue: mask ready  7 CTA wall time (thread 0)
struct WaitAcct {
  unsigned long long* w;  // [8] of this CTA, or nullptr
};
#define SAGIPS_TIMED(acct, k, expr)                                   \
  do {                                                                \
    if ((acct).w) {                                                   \
      const unsigned long long t0_ = globaltimer();                   \
      expr;                                                           \
      atomicAdd((acct).w + (k), globaltimer() - t0_);                 \
    } else {                                                          \
      expr;                                                           \
    }                                                                 \
  } while (0)

template <int N>
__device__ __forceinline__ void bulk_wait_groups() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace

namespace {
__device__ __forceinline__ int64_t ring_slot(const Ring& r, int64_t t) { return r.slots ? t % r.slots : t; }

// producer side: is the slot of tile t free right now?
__device__ __forceinline__ bool ring_slot_free(const Ring& r, int64_t t) {
  return !r.slots || t < (int64_t)r.slots || ld_relaxed(r.done + (t - r.slots)) >= r.done_target;
}
// producer side: wait until tile t may be written (slot free); whole warp
__device__ __forceinline__ void ring_acquire_slot(const Ring& r, int64_t t, int lane, WaitAcct wa = {}) {
  if (r.slots && t >= (int64_t)r.slots) {
    if (lane == 0) {
      SAGIPS_TIMED(wa, 4, wait_flag(r.done + (t - r.slots), r.done_target));
      fence_proxy_async_global();
    }
    __syncwarp();
  }
}
// producer side: publish tile `pend` once its bulk stores are complete.
// kKeep = bulk groups of later tiles that may stay in flight.
// (inc: this warp's share of the kEW completions that make a tile ready)
template <int kKeep>
__device__ __forceinline__ void ring_publish(const Ring& r, int64_t pend, int lane, uint32_t inc = 1) {
  if (r.rdy && pend >= 0 && lane == 0) {
    bulk_wait_groups<kKeep>();
    fence_proxy_async_global();
    red_release_add(r.rdy + pend, inc);
  }
}
// consumer side (single thread): wait for tile t, then order later async-proxy reads
__device__ __forceinline__ void ring_wait_ready(const Ring& r, int64_t t, WaitAcct wa = {}) {
  if (r.rdy) {
    SAGIPS_TIMED(wa, 0, wait_flag(r.rdy + t, kEW));
    fence_proxy_async_global();
  }
}
__device__ __forceinline__ void ring_consumed(const Ring& r, int64_t t) {
  if (r.done) red_release_add(r.done + t, 1);
}

}  // namespace

// ============================================================== forward
// Body of one forward layer role.  This CTA is number j of n CTAs of the
// role and processes tiles j, j + n, j + 2n, ...
template <bool kSplit, bool kFirst, bool kHead>
__device__ __forceinline__ void fwd_body(const FwdLaunch& a, int j, int n, unsigned long long* trace,
                                         WaitAcct wa = {}) {
  constexpr int P = kSplit ? 2 : 1;
  constexpr uint32_t TB = P * kPlane;
  extern __shared__ __align__(1024) uint8_t smem[];
  // first layer: two whole-tile operand stages (SIMT-produced) + one 4 KiB
  // staging buffer per epilogue warp; other layers: a FIFO of 3 operand
  // plane slots (the lo plane is consumed first and frees early) + two
  // staging buffers per epilogue warp (no wait for the bulk engine's reads)
  constexpr bool kFifo = !kFirst || kFirstFifo;
  constexpr uint32_t kRegion = 3 * kPlane + 2 * kEW * kStg;  // >= 2 TB + kEW kStg
  static_assert(kRegion >= 2 * TB + kEW * kStg, "fwd region");
  uint8_t* sW = smem;
  uint8_t* sA = sW + TB;                                  // stages / plane slots
  uint8_t* sStg = sA + (kFifo ? 3 * kPlane : 2 * TB);    // staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + kRegion);
  uint64_t* full = bars;          // [3] (first: [2] stages; FIFO: plane slots)
  uint64_t* empty = bars + 3;     // [3]
  uint64_t* tfull = bars + 6;     // [2]
  uint64_t* tempty = bars + 8;    // [2]
  double* sloss = reinterpret_cast<double*>(bars + 10);  // [8]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sloss + 8);
  int* sTile = reinterpret_cast<int*>(tmem_slot + 4);      // [8] dynamic schedule: tile of local iteration i (i % 8)
  float* sbias = reinterpret_cast<float*>(sTile + 8);      // [128]
  float* swh = sbias + 128;                                 // [128] (head) w
  float* swa = swh + 128;                                   // [128] (head) alpha * w
  Params0* p0 = reinterpret_cast<Params0*>(swh);            // (first; aliases swh and the 1 KiB after it)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    check_smem_alignment(smem);
    for (int i = 0; i < 3; ++i) {
      // first layer: H_1 rows 0-63 by the producer warps, 64-127 by the epilogue warps
      mbar_init(&full[i], kFirst ? 32 * (kPW + (a.first_help ? kEW : 0)) : 1);
      mbar_init(&empty[i], (kFirst && a.h1.base) ? 2 : 1);  // + the H_1 hi-plane store's read (lo: immediate)
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * (kHead ? kEW / 2 : kEW));  // head: 4 warps per tile (see the epilogue)
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  for (int i = tid; i < 128; i += kThreads) {
    sbias[i] = a.bias[i];
    if (kHead) {
      swh[i] = a.w_head[i];
      swa[i] = a.alpha * a.w_head[i];
    }
    if (kFirst) {
      p0->w0x[i] = a.W0[2 * i];
      p0->w0y[i] = a.W0[2 * i + 1];
      p0->b0[i] = a.b0[i];
    }
  }
  if (warp < kPW) stage_weights<kSplit>(a.W, smem_u32(sW), smem_u32(sW + kPlane), warp, lane);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > j ? (int)((ntiles - 1 - j) / n + 1) : 0;
  auto tile_of = [&](int i) { return (int64_t)j + (int64_t)i * n; };
  // dynamic tile schedule (middle layers, per-layer kernels): the loader takes
  // tiles from a global counter and passes their ids through sTile; a tile's
  // output does not depend on which CTA computes it (no per-CTA partials)
  const bool dyn = kFifo && !kFirst && !kHead && a.tile_ctr != nullptr;
  // plane FIFO: tile i's planes are p = P i (lo, split) and P i + P - 1 (hi), slot p % 3
  auto slot_lo = [&](int i) { return (P * i) % 3; };
  auto slot_hi = [&](int i) { return (P * i + P - 1) % 3; };
  auto use_lo = [&](int i) { return (P * i) / 3; };
  auto use_hi = [&](int i) { return (P * i + P - 1) / 3; };
  // first layer: wait for tile i's operand space, write its H_1 rows, signal it
  // (nrows: std::integral_constant, 16 for the producer warps, 8 for the helpers)
  auto produce_rows = [&](int i, float2 xr, bool ok, int row0, auto nrows) {
    constexpr int kRows = decltype(nrows)::value;
    if (kFifo) {
      const int sl = slot_lo(i), sh = slot_hi(i);
      if (kSplit) mbar_wait(&empty[sl], (use_lo(i) & 1) ^ 1);
      mbar_wait(&empty[sh], (use_hi(i) & 1) ^ 1);
      const uint32_t base = smem_u32(sA);
      produce_h1<kSplit, kRows>(xr, ok, w0_lane(p0, lane), a.alpha, base + sh * kPlane, base + sl * kPlane, row0, lane);
      fence_proxy_async_smem();
      if (kSplit) mbar_arrive(&full[sl]);
      mbar_arrive(&full[sh]);
    } else {
      const int s = i & 1;
      SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 4, mbar_wait(&empty[s], ((i >> 1) & 1) ^ 1));
      const uint32_t st = smem_u32(sA + s * TB);
      produce_h1<kSplit, kRows>(xr, ok, w0_lane(p0, lane), a.alpha, st, st + kPlane, row0, lane);
      fence_proxy_async_smem();
      mbar_arrive(&full[s]);
    }
  };

  if (warp < kPW) {
    // ---------------- SIMT producers of H_1 (first layer only)
    if (kFirst) {
      // rows 16 w .. 16 w + 15 (with helpers) or 32 w .. 32 w + 31
      const int nr = a.first_help ? 16 : 32;
      const float2* X2 = reinterpret_cast<const float2*>(a.X);
      auto load_x = [&](int i, bool& ok) {
        ok = false;
        if (i >= nmine || lane >= nr) return make_float2(0.f, 0.f);
        const int64_t r = tile_of(i) * 128 + nr * warp + lane;
        ok = r < a.rows;
        return ok ? __ldg(X2 + r) : make_float2(0.f, 0.f);
      };
      bool ok;
      float2 xr = load_x(0, ok);
      for (int i = 0; i < nmine; ++i) {
        bool ok_next;
        const float2 xn = load_x(i + 1, ok_next);
        if (a.first_help)
          produce_rows(i, xr, ok, 16 * warp, std::integral_constant<int, 16>{});
        else
          produce_rows(i, xr, ok, 32 * warp, std::integral_constant<int, 32>{});
        if (warp == 0 && lane == 0) trace_pt(trace, j, i, 0);
        xr = xn;
        ok = ok_next;
      }
    }
  } else if (warp == kLoadWarp) {
    // ---------------- bulk loader
    if (!kFirst && lane == 0) {
      for (int i = 0;; ++i) {
        int64_t t = -1;
        if (dyn) {
          t = atomicAdd(a.tile_ctr, 1u);
          if (t >= ntiles) t = -1;
        } else if (i < nmine) {
          t = tile_of(i);
        }
        if (dyn) sTile[i & 7] = (int)t;
        if (t < 0) {
          if (dyn) {  // sentinel: a plain arrival on the first plane slot of iteration i
            const int p = P * i, slot = p % 3;
            mbar_wait(&empty[slot], ((p / 3) & 1) ^ 1);
            mbar_arrive(&full[slot]);
          }
          break;
        }
        ring_wait_ready(a.in, t, wa);
        const uint8_t* src = a.in.base + ring_slot(a.in, t) * TB;
        // planes in consumption order: lo (split only), then hi; plane p -> slot p % 3
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const int p = P * i + q;
          const int slot = p % 3;
          SAGIPS_TIMED(wa, 1, mbar_wait(&empty[slot], ((p / 3) & 1) ^ 1));
          mbar_arrive_expect_tx(&full[slot], kPlane);
          bulk_g2s(smem_u32(sA) + slot * kPlane, src + ((kSplit && q == 0) ? kPlane : 0), kPlane, &full[slot]);
        }
        trace_pt(trace, j, i, 0);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
      const uint32_t bh = smem_u32(sW), bl = bh + kPlane;
      const bool store_h1 = kFirst && a.h1.base != nullptr;  // D step: H_1 planes for the layer-1 wgrad
      for (int i = 0; kFifo && (dyn || i < nmine); ++i) {
        const int b = i & 1;
        // lo plane first: Al.Wh, then Ah.Wh + Ah.Wl (bf16: Ah.W only)
        const int ph = P * i + (P - 1), sh = ph % 3;
        int64_t t = dyn ? -1 : tile_of(i);
        if (dyn) {  // the tile id is valid once the first plane slot's barrier completed
          const int p0 = P * i;
          SAGIPS_TIMED(wa, 2, mbar_wait(&full[p0 % 3], (p0 / 3) & 1));
          t = sTile[i & 7];
          if (t < 0) {  // forward the sentinel to the epilogue through the accumulator barrier
            SAGIPS_TIMED(wa, 3, mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1));
            mbar_arrive(&tfull[b]);
            break;
          }
        }
        SAGIPS_TIMED(wa, 3, mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1));
        const uint32_t d = tmem + (uint32_t)(b * 128);
        if (kSplit) {
          const int pl = P * i, sl = pl % 3;
          SAGIPS_TIMED(wa, 2, mbar_wait(&full[sl], (pl / 3) & 1));
          trace_pt(trace, j, i, 1);
          tc_fence_after();
          const uint32_t al = smem_u32(sA) + sl * kPlane;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
            mma_bf16(d, make_desc(al + off, 16, 1024), make_desc(bh + off, 16, 1024), idesc, k > 0);
          }
          mma_commit(&empty[sl]);
        }
        SAGIPS_TIMED(wa, 2, mbar_wait(&full[sh], (ph / 3) & 1));
        if (!kFirst) ring_consumed(a.in, t);  // both planes have been read from the input tensor
        if (store_h1) {  // the H_1 hi plane for the layer-1 wgrad (R28)
          bulk_s2g(a.h1.base + t * TB, smem_u32(sA) + sh * kPlane, kPlane);
          bulk_commit();
        }
        if (!kSplit) trace_pt(trace, j, i, 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(sA) + sh * kPlane;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          const uint64_t ad = make_desc(ah + off, 16, 1024);
          mma_bf16(d, ad, make_desc(bh + off, 16, 1024), idesc, (kSplit || k > 0) ? 1u : 0u);
          if (kSplit) mma_bf16(d, ad, make_desc(bl + off, 16, 1024), idesc, 1);
        }
        mma_commit(&empty[sh]);
        mma_commit(&tfull[b]);
        if (store_h1) {
          if (kSplit) mbar_arrive(&empty[slot_lo(i)]);  // (the lo plane is not stored)
          if (i > 0) {  // the previous tile's H_1 store is complete: publish it, free its hi slot
            bulk_wait_groups<1>();
            if (a.h1.rdy) {
              fence_proxy_async_global();
              red_release_add(a.h1.rdy + tile_of(i - 1), kEW);
            }
            mbar_arrive(&empty[slot_hi(i - 1)]);
          }
        }
      }
      if (kFifo && store_h1 && nmine > 0) {
        bulk_wait0();
        if (a.h1.rdy) {
          fence_proxy_async_global();
          red_release_add(a.h1.rdy + tile_of(nmine - 1), kEW);
        }
      }
      for (int i = 0; !kFifo && i < nmine; ++i) {
        const int s = i & 1, b = i & 1;
        SAGIPS_TIMED(wa, 2, mbar_wait(&full[s], (i >> 1) & 1));
        if (store_h1) {
          bulk_s2g(a.h1.base + tile_of(i) * TB, smem_u32(sA + s * TB), kPlane);  // hi plane (the wgrad reads only hi, R28)
          bulk_commit();
        }
        SAGIPS_TIMED(wa, 3, mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1));
        trace_pt(trace, j, i, 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(sA + s * TB), al = ah + kPlane;
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          mma_step<kSplit>(d, make_desc(ah + off, 16, 1024), make_desc(al + off, 16, 1024),
                           make_desc(bh + off, 16, 1024), make_desc(bl + off, 16, 1024), idesc, k > 0);
        }
        mma_commit(&empty[s]);
        mma_commit(&tfull[b]);
        if (store_h1 && i > 0) {  // the previous tile's H_1 store is complete: publish it, free its stage
          bulk_wait_groups<1>();
          if (a.h1.rdy) {
            fence_proxy_async_global();
            red_release_add(a.h1.rdy + tile_of(i - 1), kEW);
          }
          mbar_arrive(&empty[s ^ 1]);
        }
      }
      if (!kFifo && store_h1 && nmine > 0) {
        bulk_wait0();
        if (a.h1.rdy) {
          fence_proxy_async_global();
          red_release_add(a.h1.rdy + tile_of(nmine - 1), kEW);
        }
      }
    }
    __syncwarp();
  } else if (kHead) {
    // ---------------- head epilogue: warp e -> TMEM lane quarter q; the two
    // warps of a quarter take alternate tiles (h = tile parity = accumulator
    // buffer), each all 128 columns -- z needs no cross-warp exchange
    const int e = warp - kPW;
    const int q = warp & 3;
    const int h = e >> 2;
    const uint32_t stgA = smem_u32(sStg) + (2 * e) * kStg, stgB = stgA + kStg;  // hi / lo staging
    // sum over this CTA's tiles of dz * H at this warp's row positions,
    // accumulated in the free TMEM columns 256 + 128 h .. (one column block
    // per tile parity, so the two warps of a lane quarter never share one);
    // summed over the rows once, at the end
    const uint32_t gsum = tmem + 256u + (uint32_t)(128 * h) + ((uint32_t)(32 * q) << 16);
    const float2 alpha2 = make_float2(a.alpha, a.alpha);
    const float2* b2 = reinterpret_cast<const float2*>(sbias);
    const float2* w2 = reinterpret_cast<const float2*>(swh);
    const float2* wa2 = reinterpret_cast<const float2*>(swa);
    if (a.want_wgrad) {
      float zero[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) zero[k] = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st32(gsum + 32 * c, zero);
    }
    float gbacc = 0.f;
    double lacc = 0.0;
    int64_t pend = -1;
    // pass 2 of one 64-column region: G = dz * (Z > 0 ? w : alpha w) -> planes
    // (hi staging A, lo staging B; bf16: A / B alternate by region) and,
    // with the head gradient, gsum += dz * H
    auto region = [&](auto want, uint32_t acc, int rr, float dz, uint8_t* dst0) {
      const float2 dz2 = make_float2(dz, dz);
      const uint32_t stgH = (kSplit || rr == 0) ? stgA : stgB;
      if (kSplit) stage_free(lane);
      else stage_free_dbl(lane);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int c0 = 64 * rr + 32 * c;
        float v[32], ga[32];
        if constexpr (decltype(want)::value) tmem_ld32x2(acc + c0, gsum + c0, v, ga);
        else tmem_ld32(acc + c0, v);
        uint32_t hw[16], lw[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float2 z = add2(make_float2(v[2 * k], v[2 * k + 1]), b2[c0 / 2 + k]);
          if constexpr (decltype(want)::value) {
            const float2 t = mul2(z, alpha2);
            const float2 g = fma2(dz2, make_float2(fmaxf(z.x, t.x), fmaxf(z.y, t.y)), make_float2(ga[2 * k], ga[2 * k + 1]));
            ga[2 * k] = g.x;
            ga[2 * k + 1] = g.y;
          }
          const float2 w = w2[c0 / 2 + k], wa = wa2[c0 / 2 + k];
          const float2 G = mul2(dz2, make_float2(z.x > 0.f ? w.x : wa.x, z.y > 0.f ? w.y : wa.y));
          split2(G.x, G.y, hw[k], lw[k]);
        }
        stage_words(stgH, lane, c, hw);
        if (kSplit) stage_words(stgB, lane, c, lw);
        if constexpr (decltype(want)::value) tmem_st32(gsum + c0, ga);
      }
      return stgH;
    };
    for (int i = h; i < nmine; i += 2) {
      const int64_t t = tile_of(i);
      const int b = i & 1;
      const int64_t row = t * 128 + 32 * q + lane;
      const bool valid = row < a.rows;
      const int64_t slot = ring_slot(a.out, t);
      uint8_t* dst0 = a.out.base + slot * TB + q * 4096;
      {
        bool free_now = true;
        if (lane == 0) free_now = ring_slot_free(a.out, t);
        if (!__shfl_sync(0xffffffffu, free_now ? 1 : 0, 0)) {
          ring_publish<0>(a.out, pend, lane, 2);
          pend = -1;
        }
      }
      ring_acquire_slot(a.out, t, lane, lane == 0 ? wa : WaitAcct{});
      SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 5, mbar_wait(&tfull[b], (i >> 1) & 1));
      if ((e & 3) == 0 && lane == 0) trace_pt(trace, j, i, 2);  // warps 0 / 4: even / odd tiles
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * 128) + ((uint32_t)(32 * q) << 16);
      // pass 1: z = LeakyReLU(Z) . w + b over all 128 columns of this lane's row
      float2 dot2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        float v[32], u[32];
        tmem_ld32x2(acc + 32 * c, acc + 32 * (c + 1), v, u);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float* x = k < 16 ? v : u;
          const int kk = k & 15, col2 = 16 * c + k;  // column pair index
          const float2 zz = add2(make_float2(x[2 * kk], x[2 * kk + 1]), b2[col2]);
          const float2 tt = mul2(zz, alpha2);
          dot2 = fma2(make_float2(fmaxf(zz.x, tt.x), fmaxf(zz.y, tt.y)), w2[col2], dot2);
        }
      }
      const float z = (dot2.x + dot2.y) + *a.b_head;
      const float tl = (row < a.n_real) ? 1.f : a.label_rest;
      const float dz = valid ? (sigmoid_f(z) - tl) * a.scale : 0.f;
      if (valid) {
        a.logits[row] = z;
        lacc += (double)(tl * softplus_neg(z) + (1.f - tl) * softplus_neg(-z));
        gbacc += dz;
      }
#pragma unroll 1
      for (int rr = 0; rr < 2; ++rr) {
        const uint32_t stgH = a.want_wgrad ? region(std::true_type{}, acc, rr, dz, dst0)
                                           : region(std::false_type{}, acc, rr, dz, dst0);
        if (rr == 1) {
          tc_fence_before();
          mbar_arrive(&tempty[b]);
          if ((e & 3) == 0 && lane == 0) trace_pt(trace, j, i, 3);
        }
        flush_stage(stgH, dst0 + rr * 16384, lane);
        if (kSplit) flush_stage(stgB, dst0 + rr * 16384 + kPlane, lane);
      }
      ring_publish<2 * P>(a.out, pend, lane, 2);  // the previous tile's stores are complete (4 warps x 2)
      pend = t;
    }
    // this warp's head-gradient partial: the column sums over its 32 rows
    float gacc[4] = {0.f, 0.f, 0.f, 0.f};  // columns 32c + lane
    if (a.want_wgrad) {
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float g[32];
        tmem_ld32(gsum + 32 * c, g);
        gacc[c] = colsum32(g, lane);
      }
    }
    if (lane == 0) bulk_wait0();
    ring_publish<0>(a.out, pend, lane, 2);
    // per-CTA partials: the 8 warps' head gradients summed in shared memory
    // (the staging area is free now) in warp order; loss in fp64
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
      gbacc += __shfl_xor_sync(0xffffffffu, gbacc, w);
      lacc += __shfl_xor_sync(0xffffffffu, lacc, w);
    }
    float* sred = reinterpret_cast<float*>(sStg);  // [8][129]
    epi_sync();  // every warp is done with its staging (its bulk stores have completed)
    if (a.want_wgrad) {
#pragma unroll
      for (int c = 0; c < 4; ++c) sred[e * 129 + 32 * c + lane] = gacc[c];
      if (lane == 0) sred[e * 129 + 128] = gbacc;
    }
    if (lane == 0) sloss[e] = lacc;
    epi_sync();
    if (a.want_wgrad && e < 5) {
      for (int k = 32 * e + lane; k < 129 && k < 32 * (e + 1); k += 32) {
        float v = 0.f;
        for (int w = 0; w < kEW; ++w) v += sred[w * 129 + k];
        a.part_head[(int64_t)j * 129 + k] = v;
      }
    }
    if (e == 0 && lane == 0) {
      double sum = 0.0;
      for (int k = 0; k < kEW; ++k) sum += sloss[k];
      a.loss_part[j] = sum;
    }
  } else {
    // ---------------- epilogue: warp e -> TMEM lane quarter q, column half h
    const int e = warp - kPW;
    const int q = warp & 3;
    const int h = e >> 2;
    const int cb = 64 * h;
    // staging: first layer one buffer per warp; others hi / lo double buffers
    const uint32_t stgA = smem_u32(sStg) + (kFifo ? 2 * e : e) * kStg, stgB = kFifo ? stgA + kStg : stgA;
    int64_t pend = -1;            // tile whose stores are in flight, not yet published
    // first layer: this warp also produces H_1 rows 64 + 8e .. 64 + 8e + 7 of
    // the tile two ahead (the producer warps do rows 0-63): the stage of tile
    // i + 2 is free once the MMAs of tile i -- whose accumulator this warp
    // has just read -- are done
    const float2* X2 = reinterpret_cast<const float2*>(a.X);
    const bool helping = kFirst && a.first_help;
    auto help_x = [&](int i, bool& ok) {
      ok = false;
      if (!helping || i >= nmine || lane >= 8) return make_float2(0.f, 0.f);
      const int64_t r = tile_of(i) * 128 + 64 + 8 * e + lane;
      ok = r < a.rows;
      return ok ? __ldg(X2 + r) : make_float2(0.f, 0.f);
    };
    auto help = [&](int i, float2 xr, bool ok) {
      if (!helping || i >= nmine) return;
      produce_rows(i, xr, ok, 64 + 8 * e, std::integral_constant<int, 8>{});
    };
    if (kFirst) {
      bool ok0, ok1;
      const float2 x0 = help_x(0, ok0), x1 = help_x(1, ok1);
      help(0, x0, ok0);
      help(1, x1, ok1);
    }
    for (int i = 0; dyn || i < nmine; ++i) {
      const int b = i & 1;
      int64_t t;
      if (dyn) {  // tile id known once the accumulator is full (a sentinel ends the loop)
        SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 5, mbar_wait(&tfull[b], (i >> 1) & 1));
        t = sTile[i & 7];
        if (t < 0) break;
      } else {
        t = tile_of(i);
      }
      const int64_t row = t * 128 + 32 * q + lane;
      const bool valid = row < a.rows;
      const int64_t slot = ring_slot(a.out, t);
      uint8_t* dst = a.out.base + slot * TB + h * 16384 + q * 4096;
      bool hok = false;
      const float2 hx = help_x(i + 2, hok);  // in flight during this tile's epilogue
      // the previous tile is published after this tile's stores are issued
      // (its own stores have completed by then), unless this tile has to
      // wait for a free output slot: then publish first, or ring back-pressure
      // would feed into the pipeline latency
      {
        bool free_now = true;
        if (lane == 0) free_now = ring_slot_free(a.out, t);
        if (!__shfl_sync(0xffffffffu, free_now ? 1 : 0, 0)) {
          ring_publish<0>(a.out, pend, lane);
          pend = -1;
        }
      }
      ring_acquire_slot(a.out, t, lane, lane == 0 ? wa : WaitAcct{});
      if (!dyn) SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 5, mbar_wait(&tfull[b], (i >> 1) & 1));
      if (e == 0 && lane == 0) trace_pt(trace, j, i, 2);
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * 128 + cb) + ((uint32_t)(32 * q) << 16);
      uint32_t lo[32];
      // hi staging buffer: A (split: lo goes to B); bf16 alternates A / B by tile
      const uint32_t stgH = (kSplit || !(i & 1)) ? stgA : stgB;
      if (kFifo) stage_free_dbl(lane);
      else stage_free(lane);
      uint32_t mb[2];
      const float2 alpha2 = make_float2(a.alpha, a.alpha);
      const bool full_tile = (t + 1) * 128 <= a.rows;  // warp-uniform: only a ragged last tile has rows past the end
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float v[32];
        tmem_ld32(acc + 32 * c, v);
        const float2* b2 = reinterpret_cast<const float2*>(sbias + cb + 32 * c);
        uint32_t hw[16], m = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {  // Z = acc + b, H = LeakyReLU(Z), pairwise
          lrelu_split2(add2(make_float2(v[2 * k], v[2 * k + 1]), b2[k]), alpha2, hw[k], lo[16 * c + k]);
          m |= pos_bits(hw[k], k);
        }
        if (!full_tile && !valid) {  // rows past the end are zeros
#pragma unroll
          for (int k = 0; k < 16; ++k) hw[k] = lo[16 * c + k] = 0u;
          m = 0u;
        }
        mb[c] = m;
        stage_words(stgH, lane, c, hw);
      }
      tc_fence_before();
      mbar_arrive(&tempty[b]);
      if (e == 0 && lane == 0) trace_pt(trace, j, i, 3);
      // mask stores, then flush_stage's __syncwarp orders them before lane
      // 0's later release of this tile
      reinterpret_cast<uint2*>(a.out.mask + slot * 128 + 32 * q + lane)[h] = make_uint2(mb[0], mb[1]);
      flush_stage(stgH, dst, lane);
      if (kSplit) {
        if (kFifo) stage_free_dbl(lane);
        else stage_free(lane);
        stage_words(stgB, lane, 0, lo);
        stage_words(stgB, lane, 1, lo + 16);
        flush_stage(stgB, dst + kPlane, lane);
      }
      ring_publish<P>(a.out, pend, lane);  // the previous tile's stores are complete
      pend = t;
      help(i + 2, hx, hok);
    }
    if (lane == 0) bulk_wait0();
    ring_publish<0>(a.out, pend, lane);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================== backward
// kH1Load (first layer, wgrad): the H_1 planes are bulk-loaded (written by the
// pipelined forward first-layer role) instead of recomputed by SIMT producers
template <bool kSplit, bool kFirst, bool kWgrad, bool kH1Load = false, bool kGenG = false>
__device__ __forceinline__ void bwd_body(const BwdLaunch& a, int j, int n, unsigned long long* trace,
                                         WaitAcct wa = {}) {
  // kGenG (fused D step, the layer after the head, split): the G_4 planes are
  // not loaded but generated in shared memory by the producer warps from what
  // k_dfwd stored instead -- dz per row and the sign mask of Z_4:
  // G_4[r][c] = dz_r (Z_4[r][c] > 0 ? w_c : alpha w_c), 20 B/row instead of a
  // 512 B/row plane pair in HBM (written once, read once)
  static_assert(!kGenG || (!kFirst && kWgrad), "kGenG: non-first wgrad pass");
  constexpr int P = kSplit ? 2 : 1;
  constexpr uint32_t TB = P * kPlane;
  constexpr bool kDy = kFirst && !kWgrad;
  // kPR (wgrad, split): operands move as 32 KiB planes through plane slots
  // with their own barriers, so the next tile's planes load while this
  // tile's MMAs run (see the MMA issuer for the order)
  constexpr bool kLoadH = kWgrad && (!kFirst || kH1Load);  // H planes come from global memory
  // (split wgrad passes; the layer-1 H_1 hi plane is either bulk-loaded,
  // kH1Load, or recomputed from X by the SIMT producers into its plane slot)
  // kT (D step, first layer, plane ring; both precisions, except the bf16
  // pipelined role): the dgrad computes G_1^T (A = W_1 MN-major, B = G_2
  // K-major), so TMEM lane = channel c and column = row: dW_0 = G_1^T X and
  // db_0 accumulate per thread over rows (no shuffles), with the tile's X
  // rows bulk-loaded into shared memory
  constexpr bool kT = kFirst && kWgrad && (kSplit || !kH1Load);
  constexpr bool kPR = (kSplit && kWgrad) || kT;
  constexpr int NP = kSplit ? 3 : 2;  // kT planes per tile: Gh (, Gl), Hh
  // operand area from sG: kT 5 plane slots (its staging area is free: no G_l
  // output); otherwise two stages and the epilogue staging
  // (bf16 kGenG: a second G stage after the staging, see g_stage; the
  // allocation, bwd_smem, always has room for kT's five plane slots.  The
  // loader-fed bf16 passes are at their HBM floor: a second stage there
  // measured 2% slower at C5)
  constexpr bool kG2 = kGenG && !kSplit;
  constexpr uint32_t kSlotArea = kT ? 5 * kPlane : (kG2 ? 3 * TB : 2 * TB) + kEW * kStg;
  static_assert(kSlotArea <= 5 * kPlane || !kG2, "bf16 kGenG: room for a second G stage");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sW = smem;
  uint8_t* sG = sW + TB;     // G stage 0 (kPR: plane slots 0, 1)
  uint8_t* sH = sG + TB;     // H stage (wgrad) or G stage 1 (kPR: plane slots 2, 3)
  uint8_t* sStg = sH + TB;   // 8 x 4 KiB (dy: the partial-dot exchange; kPR first: plane slot 4)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sG + kSlotArea);
  uint64_t* fullG = bars;       // [2]
  uint64_t* emptyG = bars + 2;  // [2]
  uint64_t* fullH = bars + 4;   // [1]
  uint64_t* emptyH = bars + 5;  // [1]
  uint64_t* tfull = bars + 6;   // [2]
  uint64_t* tempty = bars + 8;  // [2]
  uint64_t* wdone = bars + 10;  // [1]
  uint64_t* pfull = bars + 12;  // [5] (kPR)
  uint64_t* pempty = bars + 17; // [5] (kPR)
  uint64_t* xfull = bars + 22;  // [2] (kT) loader -> epilogue: X rows of a tile in sX
  uint64_t* xempty = bars + 24; // [2] (kT) epilogue -> loader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 26);
  uint32_t* sOnes = tmem_slot + 4;                           // 512 B of bf16 1.0 (db MMA operand)
  Params0* p0 = reinterpret_cast<Params0*>(sOnes + 128);    // (first)
  float2* sX = reinterpret_cast<float2*>(p0);               // (kT) [2][128] X rows, overlays p0 .. tidbar
  int* sTile = reinterpret_cast<int*>(p0 + 1);              // [8] dynamic schedule: tile of local iteration i
  uint64_t* tidbar = reinterpret_cast<uint64_t*>(sTile + 8); // [8] loader -> epilogue: sTile[i % 8] written

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    check_smem_alignment(smem);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&fullG[i], 1);
      mbar_init(&emptyG[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEW);
    }
    mbar_init(&fullH[0], kLoadH ? 1 : 32 * kPW);
    mbar_init(&emptyH[0], 1);
    mbar_init(&wdone[0], 1);
    for (int k = 0; k < 8; ++k) mbar_init(&tidbar[k], 1);
    for (int k = 0; k < 2; ++k) {
      mbar_init(&xfull[k], 1);
      mbar_init(&xempty[k], 32 * kEW);
    }
    for (int k = 0; k < 5; ++k) {
      mbar_init(&pfull[k], 1);
      mbar_init(&pempty[k], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  for (int i = tid; i < 128; i += kThreads) sOnes[i] = 0x3F803F80u;
  if (kFirst && !kT) {
    for (int i = tid; i < 128; i += kThreads) {
      p0->w0x[i] = a.W0[2 * i];
      p0->w0y[i] = a.W0[2 * i + 1];
      p0->b0[i] = a.b0[i];
    }
  }
  if (kGenG) {  // the head weights w and alpha w (p0 is free: not the first layer)
    for (int i = tid; i < 128; i += kThreads) {
      p0->w0x[i] = a.gen_w[i];
      p0->w0y[i] = a.alpha * a.gen_w[i];
    }
  }
  if (warp < kPW) stage_weights<kSplit>(a.W, smem_u32(sW), smem_u32(sW + kPlane), warp, lane);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc_w = tmem + 256, acc_b = tmem + 384;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > j ? (int)((ntiles - 1 - j) / n + 1) : 0;
  auto tile_of = [&](int i) { return (int64_t)j + (int64_t)i * n; };
  // G stage of tile i: wgrad -> single stage; else a ring of 2 (sG, sH)
  // bf16 kGenG (the H plane has sH): a second G stage past the staging, so
  // tile i+1's G is generated during tile i's MMAs
  uint8_t* sG2 = sStg + kEW * kStg;
  auto g_stage = [&](int i) -> uint8_t* { return (i & 1) ? (kG2 ? sG2 : (!kWgrad ? sH : sG)) : sG; };
  // stage / parity of tile i's G: one stage for the loader-fed wgrad pass, two otherwise
  auto g_s = [&](int i) { return (kWgrad && !kG2) ? 0 : (i & 1); };
  auto g_par = [&](int i) -> uint32_t { return (kWgrad && !kG2) ? (i & 1) : ((i >> 1) & 1); };
  // dynamic tile schedule (G step: no per-CTA partial sums): the loader takes
  // tiles from a global counter; MMA warp reads ids after the stage barrier,
  // the epilogue after tidbar (so its mask loads are issued early)
  const bool dyn = !kWgrad && a.tile_ctr != nullptr;
  // kPR plane slots {slot, use}: use = how many times the slot was filled
  // before.  Three planes per tile, Gh, Hh, Gl (the wgrad reads only the hi
  // plane of H, R28), in a FIFO over slots 0-3 (plane p = 3i + k -> slot
  // p % 4); the MMA order releases them in the same order.
  struct PS {
    int slot, use;
  };
  // kT: planes Gh, Gl, Hh over 5 slots (its staging area is the 5th; every
  // plane is held until the end of its tile's MMAs, see the MMA issuer)
  constexpr int kSlots = kT ? 5 : 4;
  constexpr int kNP = kT ? NP : 3;
  auto pl_of = [&](int i, int k) -> PS { return PS{(kNP * i + k) % kSlots, (kNP * i + k) / kSlots}; };
  auto pl_gh = [&](int i) -> PS { return pl_of(i, 0); };
  auto pl_hh = [&](int i) -> PS { return pl_of(i, kT ? kNP - 1 : 1); };
  auto pl_gl = [&](int i) -> PS { return pl_of(i, kT ? 1 : 2); };  // (split only)
  auto pl_addr = [&](int slot) -> uint32_t { return smem_u32(sG) + (uint32_t)slot * kPlane; };

  if (warp < kPW) {
    // ---------------- SIMT producers of the G_4 planes (kGenG): thread = row
    if (kGenG) {
      const int r = 32 * warp + lane;
      // dz and the mask of the next tile are loaded one tile ahead (their
      // HBM latency is otherwise paid by every tile's generation)
      float dz_n = 0.f;
      uint4 mq_n = make_uint4(0u, 0u, 0u, 0u);
      if (nmine > 0) {
        dz_n = __ldg(a.gen_dz + tile_of(0) * 128 + r);
        mq_n = __ldg(a.gen_mask + tile_of(0) * 128 + r);
      }
      for (int i = 0; i < nmine; ++i) {
        const float dz = dz_n;
        const uint4 mq = mq_n;
        if (i + 1 < nmine) {
          dz_n = __ldg(a.gen_dz + tile_of(i + 1) * 128 + r);
          mq_n = __ldg(a.gen_mask + tile_of(i + 1) * 128 + r);
        }
        // the Gh plane goes to its slot as soon as it is free (it is needed
        // first); the Gl plane when the previous tile releases its slot
        // (plane FIFO: Gh, Hh, Gl).  Each pass computes G_4 = dz (w or alpha
        // w) and its split afresh: no lo words held across the wait, and a
        // rolled 32-column loop keeps the kernel's code small
        const float2 dz2 = make_float2(dz, dz);
        auto gen_plane = [&](uint32_t base, bool lo_plane) {
#pragma unroll 1
          for (int cb = 0; cb < 4; ++cb) {  // 32-column blocks: mask word cb (bit k = column 2k, bit 16 + k = 2k + 1)
            const uint32_t m = cb == 0 ? mq.x : cb == 1 ? mq.y : cb == 2 ? mq.z : mq.w;
            uint32_t hw[16], lw[16];
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              const int col = 32 * cb + 2 * kk;
              const float2 w = *reinterpret_cast<const float2*>(&p0->w0x[col]);
              const float2 wa2 = *reinterpret_cast<const float2*>(&p0->w0y[col]);
              const float2 g = mul2(dz2, make_float2(((m >> kk) & 1u) ? w.x : wa2.x, ((m >> (16 + kk)) & 1u) ? w.y : wa2.y));
              split2(g.x, g.y, hw[kk], lw[kk]);
            }
            const uint32_t* v = lo_plane ? lw : hw;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
              sts128(base + sw128_chunk(r, 4 * cb + jj, 128), v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
          }
        };
        if constexpr (kSplit) {
          const PS gh = pl_gh(i), gl = pl_gl(i);
          SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 4, mbar_wait(&pempty[gh.slot], (gh.use & 1) ^ 1));
          gen_plane(pl_addr(gh.slot), false);
          fence_proxy_async_smem();
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kPW) : "memory");
          if (warp == 0 && lane == 0) mbar_arrive(&pfull[gh.slot]);
          SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 4, mbar_wait(&pempty[gl.slot], (gl.use & 1) ^ 1));
          gen_plane(pl_addr(gl.slot), true);
          fence_proxy_async_smem();
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kPW) : "memory");
          if (warp == 0 && lane == 0) mbar_arrive(&pfull[gl.slot]);
        } else {  // bf16: the hi plane into G stage i % 2, in place of the loader's copy
          const int gs = i & 1;
          SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 4, mbar_wait(&emptyG[gs], ((i >> 1) & 1) ^ 1));
          gen_plane(smem_u32(g_stage(i)), false);
          fence_proxy_async_smem();
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kPW) : "memory");
          if (warp == 0 && lane == 0) mbar_arrive(&fullG[gs]);
        }
      }
    }
    // ---------------- SIMT producers of H_1 planes (first layer, wgrad)
    if (kFirst && kWgrad && !kH1Load) {
      const float2* X2 = reinterpret_cast<const float2*>(a.X);
      auto load_x = [&](int i, bool& ok) {
        ok = false;
        if (i >= nmine) return make_float2(0.f, 0.f);
        const int64_t r = tile_of(i) * 128 + 32 * warp + lane;
        ok = r < a.rows;
        return ok ? __ldg(X2 + r) : make_float2(0.f, 0.f);
      };
      bool ok;
      float2 xr = load_x(0, ok);
      // kT: sX overlays the shared Params0, so W_0 comes from global memory
      // (held in registers); otherwise from the shared copy, per tile
      W0Lane w0g;
      if (kT) w0g = w0_lane(a.W0, a.b0, lane);
      for (int i = 0; i < nmine; ++i) {
        bool ok_next;
        const float2 xn = load_x(i + 1, ok_next);
        if (kPR) {
          // the H_1 hi plane (all the wgrad reads, R28) into its FIFO slot;
          // the 4 producer warps meet at a named barrier, one thread arrives
          const PS ph = pl_hh(i);
          SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 4, mbar_wait(&pempty[ph.slot], (ph.use & 1) ^ 1));
          produce_h1<false, 32>(xr, ok, w0g, a.alpha, pl_addr(ph.slot), 0u, 32 * warp, lane);
          fence_proxy_async_smem();
          asm volatile("bar.sync 2, %0;" ::"n"(32 * kPW) : "memory");
          if (warp == 0 && lane == 0) mbar_arrive(&pfull[ph.slot]);
        } else {
          mbar_wait(&emptyH[0], (i & 1) ^ 1);
          produce_h1<kSplit, 32>(xr, ok, w0_lane(p0, lane), a.alpha, smem_u32(sH), smem_u32(sH) + kPlane, 32 * warp,
                                 lane);
          fence_proxy_async_smem();
          mbar_arrive(&fullH[0]);
        }
        xr = xn;
        ok = ok_next;
      }
    }
  } else if (warp == kLoadWarp) {
    // ---------------- bulk loader
    if (kPR && lane == 0) {
      auto load = [&](PS ps, const uint8_t* src) {
        SAGIPS_TIMED(wa, 1, mbar_wait(&pempty[ps.slot], (ps.use & 1) ^ 1));
        mbar_arrive_expect_tx(&pfull[ps.slot], kPlane);
        bulk_g2s(pl_addr(ps.slot), src, kPlane, &pfull[ps.slot]);
      };
      // no L2 prefetch: the plane ring issues each load a tile ahead, and
      // prefetched lines were evicted before use (ncu: +33% DRAM reads)
      for (int i = 0; i < nmine; ++i) {
        const int64_t t = tile_of(i);
        const uint8_t* gsrc = a.g.base + ring_slot(a.g, t) * TB;
        if (kT) {  // the tile's X rows (1 KiB; the epilogue zeroes rows past the end)
          const int xb = i & 1;
          mbar_wait(&xempty[xb], ((i >> 1) & 1) ^ 1);
          const int64_t r0 = t * 128;
          const uint32_t bytes = (uint32_t)((min((int64_t)128, a.rows - r0) * 8 + 15) & ~15);
          mbar_arrive_expect_tx(&xfull[xb], bytes);
          bulk_g2s(smem_u32(sX + xb * 128), reinterpret_cast<const float2*>(a.X) + r0, bytes, &xfull[xb]);
        }
        if (!kGenG) {
          ring_wait_ready(a.g, t, wa);
          load(pl_gh(i), gsrc);
        }
        if (kT && kSplit) load(pl_gl(i), gsrc + kPlane);
        if (kLoadH) {  // (else the producers write it)
          const uint8_t* hsrc = a.h.base + ring_slot(a.h, t) * TB;
          ring_wait_ready(a.h, t, wa);
          load(pl_hh(i), hsrc);
        }
        if (!kT && !kGenG) load(pl_gl(i), gsrc + kPlane);
        trace_pt(trace, j, i, 0);
      }
    } else if (!kPR && lane == 0) {
      for (int i = 0; dyn || i < nmine; ++i) {
        int64_t t = -1;
        if (dyn) {
          t = atomicAdd(a.tile_ctr, 1u);
          if (t >= ntiles) t = -1;
          sTile[i & 7] = (int)t;
          mbar_arrive(&tidbar[i & 7]);
          if (t < 0) {  // sentinel to the MMA warp through the stage barrier
            const int s = i & 1;
            mbar_wait(&emptyG[s], ((i >> 1) & 1) ^ 1);
            mbar_arrive(&fullG[s]);
            break;
          }
        } else {
          t = tile_of(i);
        }
        if (!dyn && i + 1 < nmine) {
          if (!kGenG && !a.g.slots) prefetch_l2(a.g.base + tile_of(i + 1) * TB, TB);
          if (kWgrad && !kFirst && !a.h.slots) prefetch_l2(a.h.base + tile_of(i + 1) * TB, TB);
        }
        if (kLoadH) {
          ring_wait_ready(a.h, t, wa);
          SAGIPS_TIMED(wa, 1, mbar_wait(&emptyH[0], (i & 1) ^ 1));
          mbar_arrive_expect_tx(&fullH[0], TB);
          bulk_g2s(smem_u32(sH), a.h.base + ring_slot(a.h, t) * TB, TB, &fullH[0]);
        }
        if (!kGenG) {  // (kGenG: the producers write the G stage)
          const int s = g_s(i);
          const uint32_t ph = g_par(i) ^ 1u;
          ring_wait_ready(a.g, t, wa);
          SAGIPS_TIMED(wa, 1, mbar_wait(&emptyG[s], ph));
          mbar_arrive_expect_tx(&fullG[s], TB);
          bulk_g2s(smem_u32(g_stage(i)), a.g.base + ring_slot(a.g, t) * TB, TB, &fullG[s]);
        }
        trace_pt(trace, j, i, 0);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer: the whole warp runs the loop, one elected
    // lane issues each MMA (a converged warp issues an M128 N128 K16 MMA every
    // 64 cycles; one thread of a divergent warp every 84-91)
    const WaitAcct wq = lane == 0 ? wa : WaitAcct{};
    {
      constexpr uint32_t id_d = make_idesc_bf16(128, 128, 0, 1);  // A = G (K-major), B = W (MN-major)
      constexpr uint32_t id_w = make_idesc_bf16(128, 128, 1, 1);  // A = G^T, B = H (both MN-major)
      constexpr uint32_t id_b = make_idesc_bf16(128, 16, 1, 0);   // A = G^T, B = ones (K-major)
      const uint64_t ones = make_desc(smem_u32(sOnes), 128, 256, 0);  // no swizzle: any layout reads 1.0
      const uint32_t wh = smem_u32(sW), wl = wh + kPlane;
      const uint32_t hh = smem_u32(sH), hl = hh + kPlane;
      // kPR order per tile (each plane slot is released right after its last MMA):
      //  1 Gh.Hh, Gh.1 (wgrad, db)  2 dgrad Gh.Wh, Gh.Wl -> Gh free
      //  3 Gl.Hh, Gl.1 -> Hh free  4 dgrad Gl.Wh -> Gl free, accumulator full
      // kT order per tile, maximising operand reuse between consecutive MMAs
      // (the tensor pipe is bound by its shared-memory operand reads,
      // tests/tools/mma_rate.cu) and handing the accumulator to the epilogue
      // first:  1 dgrad G_1^T per K step: Wl.Gh, Wh.Gh, Wh.Gl -> accumulator
      // full  2 wgrad + db per K step: Gh^T.1, Gh^T.Hh, Gl^T.Hh, Gl^T.1 ->
      // all three planes free
      constexpr uint32_t id_dT = make_idesc_bf16(128, 128, 1, 0);  // A = W (MN-major), B = G (K-major)
      for (int i = 0; kT && !kSplit && i < nmine; ++i) {  // bf16: one G plane, W hi only
        const int64_t t = tile_of(i);
        const int b = i & 1;
        const PS gh = pl_gh(i), ph = pl_hh(i);
        const uint32_t agh = pl_addr(gh.slot), ahh = pl_addr(ph.slot);
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[gh.slot], gh.use & 1));
        if (lane == 0) ring_consumed(a.g, t);
        SAGIPS_TIMED(wq, 3, mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1));
        if (lane == 0) trace_pt(trace, j, i, 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          mma_bf16_warp(d, make_desc(wh + km, 16384, 1024), make_desc(agh + kk, 16, 1024), id_dT, k > 0);
        }
        mma_commit_warp(&tfull[b]);
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[ph.slot], ph.use & 1));
        if (kLoadH) if (lane == 0) ring_consumed(a.h, t);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048, acc0 = (i > 0 || k > 0) ? 1u : 0u;
          const uint64_t gh_k = make_desc(agh + km, 16384, 1024);
          mma_bf16_warp(acc_b, gh_k, ones, id_b, acc0);
          mma_bf16_warp(acc_w, gh_k, make_desc(ahh + km, 16384, 1024), id_w, acc0);
        }
        mma_commit_warp(&pempty[gh.slot]);
        mma_commit_warp(&pempty[ph.slot]);
      }
      for (int i = 0; kT && kSplit && i < nmine; ++i) {
        const int64_t t = tile_of(i);
        const int b = i & 1;
        const PS gh = pl_gh(i), gl = pl_gl(i), ph = pl_hh(i);
        const uint32_t agh = pl_addr(gh.slot), agl = pl_addr(gl.slot), ahh = pl_addr(ph.slot);
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[gh.slot], gh.use & 1));
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[gl.slot], gl.use & 1));
        if (lane == 0) ring_consumed(a.g, t);  // both G planes have been read
        SAGIPS_TIMED(wq, 3, mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1));
        if (lane == 0) trace_pt(trace, j, i, 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          const uint64_t gk = make_desc(agh + kk, 16, 1024), wk = make_desc(wh + km, 16384, 1024);
          mma_bf16_warp(d, make_desc(wl + km, 16384, 1024), gk, id_dT, k > 0);
          mma_bf16_warp(d, wk, gk, id_dT, 1);
          mma_bf16_warp(d, wk, make_desc(agl + kk, 16, 1024), id_dT, 1);
        }
        mma_commit_warp(&tfull[b]);
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[ph.slot], ph.use & 1));
        if (kLoadH) if (lane == 0) ring_consumed(a.h, t);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048, acc0 = (i > 0 || k > 0) ? 1u : 0u;
          const uint64_t gh_k = make_desc(agh + km, 16384, 1024), gl_k = make_desc(agl + km, 16384, 1024);
          const uint64_t hh_k = make_desc(ahh + km, 16384, 1024);
          mma_bf16_warp(acc_b, gh_k, ones, id_b, acc0);
          mma_bf16_warp(acc_w, gh_k, hh_k, id_w, acc0);
          mma_bf16_warp(acc_w, gl_k, hh_k, id_w, 1);
          mma_bf16_warp(acc_b, gl_k, ones, id_b, 1);
        }
        mma_commit_warp(&pempty[gh.slot]);
        mma_commit_warp(&pempty[gl.slot]);
        mma_commit_warp(&pempty[ph.slot]);
      }
      for (int i = 0; kPR && !kT && i < nmine; ++i) {
        const int64_t t = tile_of(i);
        const int b = i & 1;
        const PS gh = pl_gh(i), ph = pl_hh(i), gl = pl_gl(i);
        const uint32_t agh = pl_addr(gh.slot), ahh = pl_addr(ph.slot), agl = pl_addr(gl.slot);
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[gh.slot], gh.use & 1));
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[ph.slot], ph.use & 1));
        if (kLoadH) if (lane == 0) ring_consumed(a.h, t);  // the H plane has been read
        if (lane == 0) trace_pt(trace, j, i, 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048, acc0 = (i > 0 || k > 0) ? 1u : 0u;
          const uint64_t g = make_desc(agh + km, 16384, 1024);
          mma_bf16_warp(acc_w, g, make_desc(ahh + km, 16384, 1024), id_w, acc0);
          mma_bf16_warp(acc_b, g, ones, id_b, acc0);
        }
        SAGIPS_TIMED(wq, 3, mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          const uint64_t g = make_desc(agh + kk, 16, 1024);
          mma_bf16_warp(d, g, make_desc(wh + km, 16384, 1024), id_d, k > 0);
          mma_bf16_warp(d, g, make_desc(wl + km, 16384, 1024), id_d, 1);
        }
        mma_commit_warp(&pempty[gh.slot]);
        SAGIPS_TIMED(wq, 2, mbar_wait(&pfull[gl.slot], gl.use & 1));
        if (lane == 0) ring_consumed(a.g, t);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048;
          const uint64_t g = make_desc(agl + km, 16384, 1024);
          mma_bf16_warp(acc_w, g, make_desc(ahh + km, 16384, 1024), id_w, 1);
          mma_bf16_warp(acc_b, g, ones, id_b, 1);
        }
        mma_commit_warp(&pempty[ph.slot]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          mma_bf16_warp(d, make_desc(agl + kk, 16, 1024), make_desc(wh + km, 16384, 1024), id_d, 1);
        }
        mma_commit_warp(&pempty[gl.slot]);
        mma_commit_warp(&tfull[b]);
      }
      for (int i = 0; !kPR && (dyn || i < nmine); ++i) {
        const int b = i & 1;
        const int s = g_s(i);
        SAGIPS_TIMED(wq, 2, mbar_wait(&fullG[s], g_par(i)));
        const int64_t t = dyn ? (int64_t)sTile[i & 7] : tile_of(i);
        if (t < 0) break;  // sentinel (the epilogue stops at its own tidbar)
        if (lane == 0) ring_consumed(a.g, t);
        const uint32_t zh = smem_u32(g_stage(i)), zl = zh + kPlane;
        if (kWgrad) {
          mbar_wait(&fullH[0], i & 1);
          if (kLoadH) if (lane == 0) ring_consumed(a.h, t);
          if (lane == 0) trace_pt(trace, j, i, 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t km = k * 2048;  // MN-major step (16 rows)
            const uint32_t acc0 = (i > 0 || k > 0) ? 1u : 0u;
            const uint64_t gh = make_desc(zh + km, 16384, 1024), gl = make_desc(zl + km, 16384, 1024);
            mma_step_warp<kSplit>(acc_w, gh, gl, make_desc(hh + km, 16384, 1024), make_desc(hl + km, 16384, 1024), id_w,
                             acc0);
            mma_bf16_warp(acc_b, gh, ones, id_b, acc0);
            if (kSplit) mma_bf16_warp(acc_b, gl, ones, id_b, 1);
          }
          mma_commit_warp(&emptyH[0]);
        }
        SAGIPS_TIMED(wq, 3, mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1));
        if (!kWgrad) if (lane == 0) trace_pt(trace, j, i, 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32;  // K-major step (16 columns)
          const uint32_t km = k * 2048;
          // dgrad: D[rows][in] = G[rows][out] * W[out][in]
          mma_step_warp<kSplit>(d, make_desc(zh + kk, 16, 1024), make_desc(zl + kk, 16, 1024),
                           make_desc(wh + km, 16384, 1024), make_desc(wl + km, 16384, 1024), id_d, k > 0);
        }
        mma_commit_warp(&emptyG[s]);
        mma_commit_warp(&tfull[b]);
      }
      mma_commit_warp(&wdone[0]);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warp e -> TMEM lane quarter q, column half h
    const int e = warp - kPW;
    const int q = warp & 3;
    const int h = e >> 2;
    const int cb = 64 * h;
    const uint32_t stg = smem_u32(sStg) + e * kStg;
    float2* pdy = reinterpret_cast<float2*>(sStg);  // dy: [2][128] partial dots
    float s0[2] = {0.f, 0.f}, s1[2] = {0.f, 0.f}, sb[2] = {0.f, 0.f};  // layer-0 gradients
    const float2* X2 = reinterpret_cast<const float2*>(a.X);
    int64_t pend = -1;
    if (kT) {
      // thread = channel c = 32q + lane (TMEM lane); warp half h = rows 64h..64h+63
      const int c = 32 * q + lane;
      const float w0x = __ldg(a.W0 + 2 * c), w0y = __ldg(a.W0 + 2 * c + 1), b0c = __ldg(a.b0 + c);
      // sums over rows of g x_0, g x_1 (in row order) and of g (even / odd rows)
      float2 T = make_float2(0.f, 0.f), TB = make_float2(0.f, 0.f);
      for (int i = 0; i < nmine; ++i) {
        const int64_t t = tile_of(i);
        const int b = i & 1, xb = i & 1;
        SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 7, mbar_wait(&xfull[xb], (i >> 1) & 1));
        SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 5, mbar_wait(&tfull[b], (i >> 1) & 1));
        if (e == 0 && lane == 0) trace_pt(trace, j, i, 2);
        tc_fence_after();
        const float2* xs = sX + xb * 128;
        const int64_t valid_rows = a.rows - t * 128;
        // ragged last tile: rows past the end read as x = 0 (their sX bytes were not loaded)
        auto rows = [&](auto ragged) {
#pragma unroll 1
          for (int ch = 0; ch < 2; ++ch) {
            float v[32];  // G_1^T[c][rows 64h + 32ch + k] before LeakyReLU'
            tmem_ld32(tmem + (uint32_t)(b * 128 + 64 * h + 32 * ch) + ((uint32_t)(32 * q) << 16), v);
            const float4* x4 = reinterpret_cast<const float4*>(xs + 64 * h + 32 * ch);
#pragma unroll
            for (int k = 0; k < 32; k += 2) {  // rows r, r + 1
              float4 xx = x4[k / 2];
              if constexpr (decltype(ragged)::value) {
                const int r = 64 * h + 32 * ch + k;
                if (r >= valid_rows) xx.x = xx.y = 0.f;
                if (r + 1 >= valid_rows) xx.z = xx.w = 0.f;
              }
              // Z_1 recomputed exactly as the forward's producers do
              const float za = fmaf(xx.x, w0x, fmaf(xx.y, w0y, b0c));
              const float zb = fmaf(xx.z, w0x, fmaf(xx.w, w0y, b0c));
              const float2 g = mul2(make_float2(v[k], v[k + 1]),
                                    make_float2(za > 0.f ? 1.f : a.alpha, zb > 0.f ? 1.f : a.alpha));
              T = fma2(make_float2(g.x, g.x), make_float2(xx.x, xx.y), T);
              T = fma2(make_float2(g.y, g.y), make_float2(xx.z, xx.w), T);
              TB = add2(g, TB);
            }
          }
        };
        if (valid_rows >= 128) rows(std::false_type{});
        else rows(std::true_type{});
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        mbar_arrive(&xempty[xb]);
        if (e == 0 && lane == 0) trace_pt(trace, j, i, 3);
      }
      s0[0] = T.x;
      s1[0] = T.y;
      sb[0] = TB.x + TB.y;
    }
    for (int i = 0; !kT && (dyn || i < nmine); ++i) {
      int64_t t;
      if (dyn) {
        mbar_wait(&tidbar[i & 7], (i >> 3) & 1);
        t = sTile[i & 7];
        if (t < 0) break;
      } else {
        t = tile_of(i);
      }
      const int b = i & 1;
      const int64_t row = t * 128 + 32 * q + lane;
      const bool valid = row < a.rows;
      const bool full_tile = (t + 1) * 128 <= a.rows;  // warp-uniform
      uint2 mk = make_uint2(0u, 0u);
      float2 x = make_float2(0.f, 0.f);
      if (kFirst) {
        if (valid) x = __ldg(X2 + row);
      } else {
        // sign mask of H_l (written by its producer role with the H planes)
        if (a.h.rdy) {
          if (lane == 0) SAGIPS_TIMED(wa, 6, wait_flag(a.h.rdy + t, kEW));
          __syncwarp();
        }
        mk = __ldcg(reinterpret_cast<const uint2*>(a.h.mask + ring_slot(a.h, t) * 128 + 32 * q + lane) + h);
        {  // see fwd_body
          bool free_now = true;
          if (lane == 0) free_now = ring_slot_free(a.gout, t);
          if (!__shfl_sync(0xffffffffu, free_now ? 1 : 0, 0)) {
            ring_publish<0>(a.gout, pend, lane);
            pend = -1;
          }
        }
        ring_acquire_slot(a.gout, t, lane, lane == 0 ? wa : WaitAcct{});
      }
      SAGIPS_TIMED(lane == 0 ? wa : WaitAcct{}, 5, mbar_wait(&tfull[b], (i >> 1) & 1));
      if (e == 0 && lane == 0) trace_pt(trace, j, i, 2);
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * 128 + cb) + ((uint32_t)(32 * q) << 16);
      if (!kFirst) {
        const int64_t slot = ring_slot(a.gout, t);
        uint8_t* dst = a.gout.base + slot * TB + h * 16384 + q * 4096;
        uint32_t lo[32];
        stage_free(lane);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
          const uint32_t m = c ? mk.y : mk.x;
          uint32_t hw[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {  // G' = acc * LeakyReLU'(Z), pairwise (columns 2k, 2k + 1)
            const float d0 = ((m >> mask_bit(2 * k)) & 1u) ? 1.f : a.alpha;
            const float d1 = ((m >> mask_bit(2 * k + 1)) & 1u) ? 1.f : a.alpha;
            const float2 g = mul2(make_float2(v[2 * k], v[2 * k + 1]), make_float2(d0, d1));
            split2(g.x, g.y, hw[k], lo[16 * c + k]);
          }
          if (!full_tile && !valid) {  // rows past the end are zeros
#pragma unroll
            for (int k = 0; k < 16; ++k) hw[k] = lo[16 * c + k] = 0u;
          }
          stage_words(stg, lane, c, hw);
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        if (a.h.done) {  // this warp's mask reads are complete
          __syncwarp();
          if (lane == 0) red_release_add(a.h.done + t, 1);
        }
        if (e == 0 && lane == 0) trace_pt(trace, j, i, 3);
        flush_stage(stg, dst, lane);
        if (kSplit) {
          stage_free(lane);
          stage_words(stg, lane, 0, lo);
          stage_words(stg, lane, 1, lo + 16);
          flush_stage(stg, dst + kPlane, lane);
        }
        ring_publish<P>(a.gout, pend, lane);
        pend = t;
      } else {
        // G_1 = acc * LeakyReLU'(Z_1), Z_1 = x W_0^T + b_0 recomputed exactly as
        // the producers do (pairwise FFMA2 = fmaf per lane).  Rows past the
        // end need no mask: their accumulator rows are exactly 0 (G_2 rows
        // are zero there) and x = 0.
        float2 D0 = make_float2(0.f, 0.f), D1 = make_float2(0.f, 0.f);  // dy partial dots (column pairs)
        const float2 X0 = make_float2(x.x, x.x), X1 = make_float2(x.y, x.y);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
#pragma unroll
          for (int k = 0; k < 32; k += 4) {  // layer-0 parameters as float4 (broadcast) loads
            const int cc = cb + 32 * c + k;
            const float4 wx = *reinterpret_cast<const float4*>(&p0->w0x[cc]);
            const float4 wy = *reinterpret_cast<const float4*>(&p0->w0y[cc]);
            const float4 bb = *reinterpret_cast<const float4*>(&p0->b0[cc]);
            const float2 wxa = make_float2(wx.x, wx.y), wxb = make_float2(wx.z, wx.w);
            const float2 wya = make_float2(wy.x, wy.y), wyb = make_float2(wy.z, wy.w);
            const float2 za = fma2(X0, wxa, fma2(X1, wya, make_float2(bb.x, bb.y)));
            const float2 zb = fma2(X0, wxb, fma2(X1, wyb, make_float2(bb.z, bb.w)));
            const float2 ga = mul2(make_float2(v[k], v[k + 1]),
                                   make_float2(za.x > 0.f ? 1.f : a.alpha, za.y > 0.f ? 1.f : a.alpha));
            const float2 gb = mul2(make_float2(v[k + 2], v[k + 3]),
                                   make_float2(zb.x > 0.f ? 1.f : a.alpha, zb.y > 0.f ? 1.f : a.alpha));
            if (kWgrad) {
              v[k] = ga.x;
              v[k + 1] = ga.y;
              v[k + 2] = gb.x;
              v[k + 3] = gb.y;
            } else {
              D0 = fma2(gb, wxb, fma2(ga, wxa, D0));
              D1 = fma2(gb, wyb, fma2(ga, wya, D1));
            }
          }
          if (kWgrad) {
            float g[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) g[k] = v[k] * x.x;
            s0[c] += colsum32(g, lane);
#pragma unroll
            for (int k = 0; k < 32; ++k) g[k] = v[k] * x.y;
            s1[c] += colsum32(g, lane);
            sb[c] += colsum32(v, lane);
          }
        }
        const float d0 = D0.x + D0.y, d1 = D1.x + D1.y;
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        if (e == 0 && lane == 0) trace_pt(trace, j, i, 3);
        if (kDy) {
          epi_sync();  // previous tile's reads of pdy done
          pdy[h * 128 + 32 * q + lane] = make_float2(d0, d1);
          epi_sync();
          if (h == 0 && valid) {
            const float2 o = pdy[128 + 32 * q + lane];
            reinterpret_cast<float2*>(a.dy)[row] = make_float2(d0 + o.x, d1 + o.y);
          }
        }
      }
    }
    if (lane == 0) bulk_wait0();
    if (!kFirst) ring_publish<0>(a.gout, pend, lane);
    const int64_t pq = (int64_t)j * 4 + q;
    if (kWgrad && kFirst) {
      // per-CTA layer-0 partials summed in shared memory (the plane slots are
      // free now; fixed order): kT -- the two row halves of each channel;
      // otherwise the 4 lane quarters of each column
      (void)pq;
      tc_fence_before();
      epi_sync();  // all epilogue warps are past their last tile
      float* sred = reinterpret_cast<float*>(sG);  // [4][384]
      if (kT) {
        const int c = 32 * q + lane;
        sred[h * 384 + 2 * c] = s0[0];
        sred[h * 384 + 2 * c + 1] = s1[0];
        sred[h * 384 + 256 + c] = sb[0];
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int cc = cb + 32 * c + lane;
          sred[q * 384 + 2 * cc] = s0[c];
          sred[q * 384 + 2 * cc + 1] = s1[c];
          sred[q * 384 + 256 + cc] = sb[c];
        }
      }
      epi_sync();
      for (int k = e * 32 + lane; k < 384; k += 32 * kEW) {
        float v = 0.f;
        for (int qq = 0; qq < (kT ? 2 : 4); ++qq) v += sred[qq * 384 + k];
        a.part_l0[(int64_t)j * 384 + k] = v;
      }
    }
    if (kWgrad) {
      // TMEM lane = output feature o, columns = input features; warp (q, h)
      // writes rows 32q.., columns 64h..64h+63 of this CTA's partial
      const int o = 32 * q + lane;
      float* dst = a.part + (int64_t)j * 128 * 128 + (int64_t)o * 128;
      if (nmine > 0) {
        mbar_wait(&wdone[0], 0);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc_w + cb + 32 * c + ((uint32_t)(32 * q) << 16), v);
#pragma unroll
          for (int k = 0; k < 32; k += 4)
            *reinterpret_cast<float4*>(dst + cb + 32 * c + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
        }
      } else {
        for (int k = 0; k < 64; k += 4) *reinterpret_cast<float4*>(dst + cb + k) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (h == 0) {
        float v[32];
        if (nmine > 0) tmem_ld32(acc_b + ((uint32_t)(32 * q) << 16), v);
        a.part_db[(int64_t)j * 128 + o] = nmine > 0 ? v[0] : 0.f;
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

// ============================================================== kernels
// trace: per-CTA launch stamps (start, end) next to the per-tile ones, and
// (diagnostic build SAGIPS_BUILD_WAITS=1 only: the accounting costs
// registers) the CTA's summed wait times per role (slots 4 + k, k as in
// SAGIPS_TIMED: 1 loader slot, 2 MMA operands, 3 MMA accumulator, 4
// producers' slot, 5 epilogue accumulator, 6 mask flag, 7 epilogue X rows)
__device__ __forceinline__ unsigned long long* cta_stamps(unsigned long long* trace);
__device__ __forceinline__ WaitAcct cta_waits(unsigned long long* cs) {
#ifdef SAGIPS_WAIT_ACCT
  return WaitAcct{cs ? cs + 4 : nullptr};
#else
  (void)cs;
  return WaitAcct{};
#endif
}
template <bool kSplit, bool kFirst, bool kHead>
__global__ void __launch_bounds__(kThreads, 1) k_fwd(const __grid_constant__ FwdLaunch a, unsigned long long* trace) {
  unsigned long long* cs = cta_stamps(trace);
  if (cs && threadIdx.x == 0) cs[0] = globaltimer();
  fwd_body<kSplit, kFirst, kHead>(a, blockIdx.x, gridDim.x, trace, cta_waits(cs));
  if (cs && threadIdx.x == 0) cs[1] = globaltimer();
}
template <bool kSplit, bool kFirst, bool kWgrad, bool kH1Load = false, bool kGenG = false>
__global__ void __launch_bounds__(kThreads, 1) k_bwd(const __grid_constant__ BwdLaunch a, unsigned long long* trace) {
  unsigned long long* cs = cta_stamps(trace);
  if (cs && threadIdx.x == 0) cs[0] = globaltimer();
  bwd_body<kSplit, kFirst, kWgrad, kH1Load, kGenG>(a, blockIdx.x, gridDim.x, trace, cta_waits(cs));
  if (cs && threadIdx.x == 0) {
    cs[1] = globaltimer();
    unsigned int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    cs[2] = sm;
  }
}

// The whole D step (kD: wgrad, head and layer-0 gradients) or G step (dy) as
// one dataflow pipeline: CTAs are partitioned into the six layer roles (first,
// mid, head, bwd3, bwd2, bwd1), all co-resident (cooperative launch); tiles
// stream between roles through L2-resident rings.

// ============================================================== partial sums
// out[j] = sum_p part[p*ld + j], j < n: 32 outputs x 8 part groups per block
// (group g sums parts g, g+8, ... in order; the 8 group sums are added in
// order -- deterministic)
__global__ void __launch_bounds__(256) k_sum_parts(const float* __restrict__ part, int nparts, int64_t ld, int n,
                                                   float* __restrict__ out) {
  __shared__ float red[8][33];
  const int jl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + jl;
  float s = 0.f;
  if (j < n) {
#pragma unroll 4
    for (int p = g; p < nparts; p += 8) s += __ldg(part + (int64_t)p * ld + j);
  }
  red[g][jl] = s;
  __syncthreads();
  if (g == 0 && j < n) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][jl];
    out[j] = t;
  }
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
  const size_t TB = (split ? 2 : 1) * (size_t)kPlane;
  return TB + 3 * (size_t)kPlane + 2 * kEW * kStg + 10 * 8 + 8 * 8 + 16 + 32 + 4 * (128 + 128 + 256);  // tiles, bias, w_head / Params0
}
static size_t bwd_smem(bool split) {
  const size_t TB = (split ? 2 : 1) * (size_t)kPlane;
  // operand area: two stages + staging, or the first layer's 5 plane slots (kT, bf16 too)
  const size_t area = std::max<size_t>(2 * TB + kEW * kStg, 5 * (size_t)kPlane);
  return TB + area + 26 * 8 + 16 + 512 + std::max<size_t>(sizeof(Params0) + 32 + 64, 2 * 128 * 8);
}

template <typename K>
static void allow_smem(K kern, size_t bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static void configure_layers() {
  static bool done = false;
  if (done) return;
  done = true;
  static_assert(3 * 2 * kPlane + kEW * kStg + 2048 + 1024 <= kSmemLimit, "shared-memory budget");
#define SAGIPS_FWD(S, F, H) allow_smem(k_fwd<S, F, H>, fwd_smem(S));
  SAGIPS_FWD(true, true, false) SAGIPS_FWD(true, false, false) SAGIPS_FWD(true, false, true)
  SAGIPS_FWD(false, true, false) SAGIPS_FWD(false, false, false) SAGIPS_FWD(false, false, true)
#undef SAGIPS_FWD
#define SAGIPS_BWD(S, F, W) allow_smem(k_bwd<S, F, W>, bwd_smem(S));
  SAGIPS_BWD(true, false, true) SAGIPS_BWD(true, true, true) SAGIPS_BWD(true, false, false)
  SAGIPS_BWD(true, true, false) SAGIPS_BWD(false, false, true) SAGIPS_BWD(false, true, true)
  SAGIPS_BWD(false, false, false) SAGIPS_BWD(false, true, false)
#undef SAGIPS_BWD
  allow_smem(k_bwd<true, true, true, true>, bwd_smem(true));
  allow_smem(k_bwd<true, false, true, false, true>, bwd_smem(true));
  allow_smem(k_bwd<false, false, true, false, true>, bwd_smem(false));
  allow_smem(k_bwd<false, true, true, true>, bwd_smem(false));
}

__device__ unsigned long long g_trace[kTraceLaunches][kTraceCtas * kTraceTiles * 4];
// per-CTA [start, first tile staged, end] globaltimer stamps of each traced launch
__device__ unsigned long long g_ctatime[kTraceLaunches][kMaxSms][12];
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

__device__ __forceinline__ unsigned long long* cta_stamps(unsigned long long* trace) {
  if (!trace) return nullptr;
  const size_t li = (size_t)(trace - &g_trace[0][0]) / (kTraceCtas * kTraceTiles * 4);
  if (li >= (size_t)kTraceLaunches || blockIdx.x >= (unsigned)kMaxSms) return nullptr;
  return g_ctatime[li][blockIdx.x];
}

size_t tc_trace_bytes() { return sizeof(g_trace) + sizeof(g_ctatime); }
int tc_trace_copy(void* host) {
  g_trace_next = 0;
  if (cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace)) != cudaSuccess) return -1;
  return cudaMemcpyFromSymbol(static_cast<char*>(host) + sizeof(g_trace), g_ctatime, sizeof(g_ctatime)) == cudaSuccess
             ? 0 : -1;
}

// SAGIPS_SYNC=1 (debugging): synchronize after every layer launch and report
static void debug_sync(const char* what, int kind, cudaStream_t st) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SAGIPS_SYNC");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(st);
  fprintf(stderr, "[sagips] %s kind %d: %s\n", what, kind, cudaGetErrorString(e));
}

int tc_layers_grid(int64_t rows) { return (int)std::min<int64_t>(std::max<int64_t>((rows + 127) / 128, 1), sm_count()); }
size_t plane_tile_bytes(bool split) { return (split ? 2 : 1) * (size_t)kPlane; }

void launch_tc_fwd(bool split, int kind, const FwdLaunch& L, cudaStream_t st) {
  configure_layers();
  unsigned long long* tr = trace_slot();
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = fwd_smem(split);
  if (split) {
    if (kind == FWD_FIRST) k_fwd<true, true, false><<<grid, kThreads, sm, st>>>(L, tr);
    else if (kind == FWD_MID) k_fwd<true, false, false><<<grid, kThreads, sm, st>>>(L, tr);
    else k_fwd<true, false, true><<<grid, kThreads, sm, st>>>(L, tr);
  } else {
    if (kind == FWD_FIRST) k_fwd<false, true, false><<<grid, kThreads, sm, st>>>(L, tr);
    else if (kind == FWD_MID) k_fwd<false, false, false><<<grid, kThreads, sm, st>>>(L, tr);
    else k_fwd<false, false, true><<<grid, kThreads, sm, st>>>(L, tr);
  }
  count_launch();
  debug_sync("k_fwd", kind, st);
}

void launch_tc_bwd(bool split, bool first, bool wgrad, const BwdLaunch& L, cudaStream_t st) {
  configure_layers();
  unsigned long long* tr = trace_slot();
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = bwd_smem(split);
  const bool h1load = first && wgrad && L.h.base != nullptr;
#define SAGIPS_BWD_LAUNCH(S)                                                                   \
  if (!first && wgrad && L.gen_dz) k_bwd<S, false, true, false, true><<<grid, kThreads, sm, st>>>(L, tr);       \
  else if (!first && wgrad) k_bwd<S, false, true><<<grid, kThreads, sm, st>>>(L, tr);          \
  else if (h1load) k_bwd<S, true, true, true><<<grid, kThreads, sm, st>>>(L, tr);              \
  else if (first && wgrad) k_bwd<S, true, true><<<grid, kThreads, sm, st>>>(L, tr);            \
  else if (!first) k_bwd<S, false, false><<<grid, kThreads, sm, st>>>(L, tr);                  \
  else k_bwd<S, true, false><<<grid, kThreads, sm, st>>>(L, tr);
  if (split) {
    SAGIPS_BWD_LAUNCH(true)
  } else {
    SAGIPS_BWD_LAUNCH(false)
  }
#undef SAGIPS_BWD_LAUNCH
  count_launch();
  debug_sync("k_bwd", (first ? 1 : 0) + (wgrad ? 2 : 0), st);
}

// Cooperative launch (all CTAs co-resident, one per SM): returns false if the
// device cannot host the grid.

void launch_sum_parts(const float* part, int nparts, int64_t ld, int n, float* out, cudaStream_t st) {
  k_sum_parts<<<(n + 31) / 32, 256, 0, st>>>(part, nparts, ld, n, out);
  count_launch();
}

}  // namespace sagips
