// k_fused.cu -- the discriminator MLP (paper preset [2,128,128,128,128,1],
// P:297, R4) on chip: ONE persistent kernel runs every layer of a tile,
// forward and backward, without activations touching HBM.
//
// Where the data live (per CTA, one CTA per SM):
//   shared memory  the three 128 x 128 hidden-layer weights W_1..W_3 as bf16
//                  planes (hi, and lo = bf16(W - hi) for the fp32-class
//                  split, R28): 6 x 32 KiB = 192 KiB, staged once per launch;
//                  they are the B operand of every MMA -- K-major (forward,
//                  D = A W^T) and MN-major (dgrad, D = A W) views of the same
//                  bytes (tc_util.cuh SW128 layout);
//   tensor memory  two tile slots of 256 columns: the fp32 accumulator of the
//                  current layer (128 columns) and the current layer's INPUT
//                  activations as the MMA's A operand (tcgen05.mma reads A
//                  from TMEM: row m = lane m, bf16 pairs per 32-bit column;
//                  hi in 64 columns, lo in 64) -- checked on B200 by
//                  tests/tools/tmem_a_check.cu;
//   registers      the LeakyReLU' sign bits of Z_1..Z_3 (64 bits per thread
//                  and layer) for the backward.
//
// Warp roles (512 threads): warps 0-7 own tile slot 0, warps 8-15 tile slot
// 1 (warp w of a group: TMEM lane quarter w % 4, column half w / 4 -- one
// thread = one row, 64 columns).  When a group has written a layer's A
// operand it meets at a named barrier and its first warp issues that layer's
// MMAs (warp-converged, one elected lane) and commits them to the slot's
// mbarrier.  While one slot's warps run an epilogue, the tensor core runs
// the other slot's layer.  (A separate MMA warp would make 17 warps, 5 on one
// SM sub-partition, capping every thread at 96 registers.)
//
// k_gstep (a8, the G step through the updated D, R8): per 128-row
// tile of fake events Y:
//   H_1 = LReLU(Y W_0^T + b_0)                       SIMT -> TMEM A
//   Z_{l+1} = H_l W_l^T + b_l, H_{l+1} = LReLU(.)     MMA + epilogue, l = 1..3
//   z = H_4 . w + b, L_G term softplus(-z), dz = (sigmoid(z) - 1) / N
//   G_4 = dz w (.) LReLU'(Z_4)                        epilogue -> TMEM A
//   G_l = (G_{l+1} W_l) (.) LReLU'(Z_l), l = 3..1     MMA (dgrad) + epilogue
//   dy = G_1 W_0                                      epilogue -> HBM (8 B/row)
// HBM traffic: 8 B/row in (Y), 8 B/row out (dy) + 4 B (logit); the weights
// once per CTA.  Products (split): A*B ~= Ah*Bh + Ah*Bl + Al*Bh (bf16x3, fp32
// accumulation), as the per-layer kernels.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "ctx.h"
#include "tc_util.cuh"

namespace sagips {

using namespace tc;

namespace {

constexpr int kGroupWarps = 8;                      // per tile slot
constexpr int kThreadsF = 32 * 2 * kGroupWarps;     // 512
constexpr uint32_t kPlaneF = 128 * 128 * 2;         // one bf16 plane of a 128 x 128 tile

struct SmemVec {
  float b[3][128];        // biases of W_1..W_3
  float w4[128], aw4[128];  // head w, alpha w
  float w0x[128], w0y[128], b0[128];
  float xdot[2][128][2];  // per slot, per row: the two column halves' partial head dots
  float xdy[2][128][4];   // per slot, per row: the two halves' partial dy (x, y)
  float red[16 * 65];     // per-CTA partials at the end (k_dfwd head gradient)
  double loss[kThreadsF / 32];
  uint64_t acc_full[2];
  uint32_t tmem;
};

__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(uint64_t r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)), "l"(pk2(c.x, c.y)));
  return upk2(d);
}
// bf16x2 word {low half: bf16(a), high half: bf16(b)}, round to nearest even
__device__ __forceinline__ uint32_t bf16x2_rn(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
// hi = bf16(a, b), lo = bf16(a - hi, b - hi)
__device__ __forceinline__ void split2(float2 v, uint32_t& hi, uint32_t& lo) {
  hi = bf16x2_rn(v.x, v.y);
  const float2 d = sub2(v, make_float2(__uint_as_float(hi << 16), __uint_as_float(hi & 0xffff0000u)));
  lo = bf16x2_rn(d.x, d.y);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]: warp-converged, one elected lane issues
__device__ __forceinline__ void mma_ts_warp(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// L2 prefetch of a slot's next tile's input rows (experiment builds switch
// them off with build.py SAGIPS_BUILD_DEFS)
#ifdef SAGIPS_NO_XPREFETCH_G
constexpr bool kPrefetchY = false;
#else
constexpr bool kPrefetchY = true;
#endif
#ifdef SAGIPS_NO_XPREFETCH_D
constexpr bool kPrefetchX = false;
#else
constexpr bool kPrefetchX = true;
#endif

// SAGIPS_FUSED_TRACE: per-CTA stamps after the phase stamps, [kernel][256 CTAs][4]:
// kernel entry, weights staged, tile loop done, SM id (globaltimer ns)
constexpr size_t kFTracePhaseWords = 2 * 2 * 64 * 6 * 4;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cta_stamp(unsigned long long* trace, int kern, int k) {
  if (trace && threadIdx.x == 0 && blockIdx.x < 256) {
    unsigned long long* c = trace + kFTracePhaseWords + ((size_t)kern * 256 + blockIdx.x) * 4;
    c[k] = gtimer();
    if (k == 0) {
      unsigned int sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      c[3] = sm;
    }
  }
}

// L2 prefetch of rows [r0, r0 + n) of a float2 array: the bulk prefetch needs
// 16-byte aligned addresses and sizes, and the fake rows (X + 2N floats) are
// only 8-byte aligned when N is odd -- prefetch the aligned interior
__device__ __forceinline__ void prefetch_rows(const float2* base, int64_t r0, int64_t n) {
  const uintptr_t b = reinterpret_cast<uintptr_t>(base + r0);
  const uintptr_t s0 = (b + 15) & ~(uintptr_t)15, e0 = (b + (uintptr_t)n * 8) & ~(uintptr_t)15;
  if (e0 > s0) prefetch_l2(reinterpret_cast<const void*>(s0), (uint32_t)(e0 - s0));
}

// named barrier of one slot group (8 warps)
__device__ __forceinline__ void group_sync(int s) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + s), "n"(32 * kGroupWarps) : "memory");
}

// named barrier of the two warps that own one row quarter q of slot s (column
// halves h = 0, 1): the head's z / dy exchange between them needs no more
__device__ __forceinline__ void pair_sync(int s, int q) {
  asm volatile("bar.sync %0, 64;" ::"r"(3 + 4 * s + q) : "memory");
}

// W [128][128] fp32 -> hi (/ lo) planes, SW128 layout; all threads of the CTA
template <bool kSplit>
__device__ __forceinline__ void stage_w(const float* __restrict__ W, uint32_t hi, uint32_t lo) {
  for (int idx = threadIdx.x; idx < 128 * 32; idx += kThreadsF) {
    const int r = idx >> 5, c = 4 * (idx & 31);
    const float4 x = __ldg(reinterpret_cast<const float4*>(W) + idx);
    const uint32_t off = sw128_offset(r, c, 128);
    uint32_t h0, h1, l0, l1;
    split2(make_float2(x.x, x.y), h0, l0);
    split2(make_float2(x.z, x.w), h1, l1);
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(hi + off), "r"(h0), "r"(h1));
    if (kSplit) asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(lo + off), "r"(l0), "r"(l1));
  }
}


// shared-memory vector reads that stay where they are written (the compiler
// would otherwise hoist the loop-invariant parameter reads out of the tile
// loop and spill them: LDS is cheaper than LDL)
__device__ __forceinline__ float4 lds4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ float2 lds2(const float* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(smem_u32(p)));
  return v;
}

// Activation sign masks of the per-layer kernels' HBM format (16 B per row,
// 32 bits per 32-column block: column 2k is bit k, column 2k+1 bit 16 + k,
// set iff bf16(H) > 0, R30), from the packed hi word of a pair
__device__ __forceinline__ uint32_t pos_bits(uint32_t hi, int k) {
  uint32_t gt;
  asm("set.gt.u32.bf16x2 %0, %1, %2;" : "=r"(gt) : "r"(hi), "r"(0u));
  return gt & (0x00010001u << k);
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
using tc::store_plane_words;  // (tc_util.cuh: STG.256 whole-sector plane stores)

}  // namespace



// The MMAs of one layer of a tile slot: phases 0-2 forward W_1..W_3
// (D = A W^T, K-major B), 3-5 dgrad W_3..W_1 (D = A W, MN-major B); A from the
// slot's TMEM columns (hi at +128, lo at +192), accumulator at +0.  Called by
// one whole warp (warp-converged issue, one elected lane), then committed.
template <bool kSplit>
__device__ __forceinline__ void issue_layer(uint32_t acc, uint32_t wbase, int p) {
  constexpr uint32_t TBw = (kSplit ? 2 : 1) * kPlaneF;
  constexpr uint32_t idf = make_idesc_bf16(128, 128, 0, 0);  // A (TMEM, K-major) x W^T (K-major)
  constexpr uint32_t idd = make_idesc_bf16(128, 128, 0, 1);  // A (TMEM) x W (MN-major)
  const uint32_t ah = acc + 128u, al = acc + 192u;
  const int l = p < 3 ? p : 5 - p;  // weight W_{l+1}
  const uint32_t wh = wbase + l * TBw, wl = wh + kPlaneF;
  if (p < 3) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
      const uint64_t bh = make_desc(wh + off, 16, 1024);
      mma_ts_warp(acc, ah + 8 * k, bh, idf, k > 0 ? 1u : 0u);
      if (kSplit) {
        mma_ts_warp(acc, al + 8 * k, bh, idf, 1u);
        mma_ts_warp(acc, ah + 8 * k, make_desc(wl + off, 16, 1024), idf, 1u);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t off = k * 2048;
      const uint64_t bh = make_desc(wh + off, 16384, 1024);
      mma_ts_warp(acc, ah + 8 * k, bh, idd, k > 0 ? 1u : 0u);
      if (kSplit) {
        mma_ts_warp(acc, al + 8 * k, bh, idd, 1u);
        mma_ts_warp(acc, ah + 8 * k, make_desc(wl + off, 16384, 1024), idd, 1u);
      }
    }
  }
}

template <bool kSplit>
__global__ void __launch_bounds__(kThreadsF, 1) k_gstep(const __grid_constant__ GStepArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  cta_stamp(a.trace, 0, 0);
  constexpr uint32_t TBw = (kSplit ? 2 : 1) * kPlaneF;
  SmemVec* sv = reinterpret_cast<SmemVec*>(smem + 3 * TBw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (smem_u32(smem) & 1023u) __trap();
  const uint32_t wbase = smem_u32(smem);
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) mbar_init(&sv->acc_full[s], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&sv->tmem);
  for (int l = 0; l < 3; ++l) stage_w<kSplit>(a.W[l + 1], wbase + l * TBw, wbase + l * TBw + kPlaneF);
  for (int i = tid; i < 128; i += kThreadsF) {
    for (int l = 0; l < 3; ++l) sv->b[l][i] = a.b[l + 1][i];
    sv->w4[i] = a.w4[i];
    sv->aw4[i] = a.alpha * a.w4[i];
    sv->w0x[i] = a.W[0][2 * i];
    sv->w0y[i] = a.W[0][2 * i + 1];
    sv->b0[i] = a.b[0][i];
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sv->tmem;
  cta_stamp(a.trace, 0, 1);
  const int64_t ntiles = (a.rows + 127) / 128;
  const int j = blockIdx.x, n = gridDim.x;
  const int nmine = ntiles > j ? (int)((ntiles - 1 - j) / n + 1) : 0;

  // slot group s: thread = row 32 q + lane of the tile, columns 64 h .. 64 h + 63
  const int s = warp >> 3, w8 = warp & 7, q = w8 & 3, h = w8 >> 2;
  const int r = 32 * q + lane;
  const uint32_t lanes = (uint32_t)(32 * q) << 16;
  const uint32_t slot = tmem + 256u * s;
  const uint32_t accT = slot + lanes + 64u * h;          // this thread's 64 accumulator columns
  const uint32_t ahT = slot + 128u + lanes + 32u * h;    // its 32 A-hi columns (64 bf16)
  const uint32_t alT = ahT + 64u;
  const float2 alpha2 = make_float2(a.alpha, a.alpha);
  const float b4 = *a.b4;
  uint32_t acc_ph = 0;
  double lacc = 0.0;
  auto put_a = [&](int c, const uint32_t* hw, const uint32_t* lw) {
    tmem_st16(ahT + 16u * c, hw);
    if (kSplit) tmem_st16(alT + 16u * c, lw);
  };
  // the slot's A operand is complete: the group's first warp issues layer p
  int cur_i = 0;
  // diagnostic stamps (CTA 0, first thread of each group): [slot][local tile / 2][phase][4]
  auto stamp = [&](int p, int k) {
    if (a.trace && j == 0 && w8 == 0 && lane == 0 && cur_i / 2 < 64)
      a.trace[((s * 64 + cur_i / 2) * 6 + p) * 4 + k] = clock64();
  };
  auto run_layer = [&](int p) {
    stamp(p, 0);
    tmem_st_wait();
    tc_fence_before();
    group_sync(s);
    stamp(p, 1);
    if (w8 == 0) {
      tc_fence_after();
      issue_layer<kSplit>(slot, wbase, p);
      mma_commit_warp(&sv->acc_full[s]);
    }
    stamp(p, 2);
    mbar_wait(&sv->acc_full[s], acc_ph & 1u);
    ++acc_ph;
    tc_fence_after();
    stamp(p, 3);
  };
  // LeakyReLU of a pair z (max(z, alpha z) for 0 <= alpha < 1, R6), split into
  // bf16 hi / lo words, sign bits in the pos_bits layout (R30)
  auto act_pair = [&](float2 z, int k, uint32_t& hw, uint32_t& lw, uint32_t& m) {
    const float2 t = mul2(z, alpha2);
    split2(make_float2(fmaxf(z.x, t.x), fmaxf(z.y, t.y)), hw, lw);
    m |= pos_bits(hw, k);
  };
  // LeakyReLU' of columns 2k, 2k+1 from the sign bits
  auto dact_pair = [&](float2 g, uint32_t m, int k) {
    return make_float2(g.x * (((m >> k) & 1u) ? 1.f : a.alpha), g.y * (((m >> (16 + k)) & 1u) ? 1.f : a.alpha));
  };
  for (int i = s; i < nmine; i += 2) {
    cur_i = i;
    const int64_t row = (int64_t)(j + (int64_t)i * n) * 128 + r;
    const bool valid = row < a.rows;
    const float2 x = valid ? __ldg(a.Y + row) : make_float2(0.f, 0.f);
    if (kPrefetchY && w8 == 0 && lane == 0 && i + 2 < nmine) {  // this slot's next tile's rows into L2
      const int64_t r0 = (int64_t)(j + (int64_t)(i + 2) * n) * 128;
      prefetch_rows(a.Y, r0, a.rows - r0 < 128 ? a.rows - r0 : 128);
    }
    uint32_t m1[2], m2[2], m3[2];  // LeakyReLU' sign bits of Z_1..Z_3 (two 32-column chunks)
    // H_1 = LeakyReLU(fma(x0, w0x, fma(x1, w0y, b0)))  (the per-layer kernels' order)
    {
      const float2 X0 = make_float2(x.x, x.x), X1 = make_float2(x.y, x.y);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hw[16], lw[16], m = 0;
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const int col = 64 * h + 32 * c + 2 * k;
          const float4 wx = lds4(&sv->w0x[col]);
          const float4 wy = lds4(&sv->w0y[col]);
          const float4 bb = lds4(&sv->b0[col]);
          act_pair(fma2(X0, make_float2(wx.x, wx.y), fma2(X1, make_float2(wy.x, wy.y), make_float2(bb.x, bb.y))), k,
                   hw[k], lw[k], m);
          act_pair(fma2(X0, make_float2(wx.z, wx.w), fma2(X1, make_float2(wy.z, wy.w), make_float2(bb.z, bb.w))),
                   k + 1, hw[k + 1], lw[k + 1], m);
        }
        m1[c] = m;
        put_a(c, hw, lw);
      }
    }
    // forward W_1, W_2: H_{l+1} = LeakyReLU(acc + b_l)
#pragma unroll 1
    for (int l = 0; l < 2; ++l) {
      run_layer(l);
      float v[64];
      tmem_ld32x2(accT, accT + 32u, v, v + 32);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hw[16], lw[16], m = 0;
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const float4 bq = lds4(&sv->b[l][64 * h + 32 * c + 2 * k]);
          act_pair(add2(make_float2(v[32 * c + 2 * k], v[32 * c + 2 * k + 1]), make_float2(bq.x, bq.y)), k, hw[k], lw[k], m);
          act_pair(add2(make_float2(v[32 * c + 2 * k + 2], v[32 * c + 2 * k + 3]), make_float2(bq.z, bq.w)), k + 1,
                   hw[k + 1], lw[k + 1], m);
        }
        if (l == 0) m2[c] = m;
        else m3[c] = m;
        put_a(c, hw, lw);
      }
    }
    // head: Z_4 = acc + b_3, z = LeakyReLU(Z_4) . w + b, dz, G_4 = dz (Z_4 > 0 ? w : alpha w)
    {
      run_layer(2);
      float v[64];
      tmem_ld32x2(accT, accT + 32u, v, v + 32);
      uint32_t m4[2] = {0u, 0u};
      float2 dot = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int col = 64 * h + 32 * c + 2 * k;
          const float2 z = add2(make_float2(v[32 * c + 2 * k], v[32 * c + 2 * k + 1]),
                                lds2(&sv->b[2][col]));
          const float2 t = mul2(z, alpha2);
          const float2 hh = make_float2(fmaxf(z.x, t.x), fmaxf(z.y, t.y));
          dot = fma2(hh, lds2(&sv->w4[col]), dot);
          m4[c] |= pos_bits(bf16x2_rn(hh.x, hh.y), k);
        }
      }
      sv->xdot[s][r][h] = dot.x + dot.y;
      pair_sync(s, q);
      const float zz = (sv->xdot[s][r][0] + sv->xdot[s][r][1]) + b4;
      const float dz = valid ? (sigmoid_f(zz) - 1.0f) * a.scale : 0.f;
      if (valid && h == 0) {
        a.logits[row] = zz;
        lacc += (double)softplus_neg(zz);
      }
      const float2 dz2 = make_float2(dz, dz);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hw[16], lw[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int col = 64 * h + 32 * c + 2 * k;
          const float2 w = lds2(&sv->w4[col]);
          const float2 wa = lds2(&sv->aw4[col]);
          const uint32_t m = m4[c];
          split2(mul2(dz2, make_float2(((m >> k) & 1u) ? w.x : wa.x, ((m >> (16 + k)) & 1u) ? w.y : wa.y)), hw[k],
                 lw[k]);
        }
        put_a(c, hw, lw);
      }
    }
    // dgrad W_3, W_2: G_l = acc (.) LeakyReLU'(Z_l)
#pragma unroll 1
    for (int l = 0; l < 2; ++l) {
      run_layer(3 + l);
      float v[64];
      tmem_ld32x2(accT, accT + 32u, v, v + 32);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t m = (l == 0) ? m3[c] : m2[c];
        uint32_t hw[16], lw[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
          split2(dact_pair(make_float2(v[32 * c + 2 * k], v[32 * c + 2 * k + 1]), m, k), hw[k], lw[k]);
        put_a(c, hw, lw);
      }
    }
    // dgrad W_1: G_1 = acc (.) LeakyReLU'(Z_1), dy = G_1 W_0
    {
      run_layer(5);
      float v[64];
      tmem_ld32x2(accT, accT + 32u, v, v + 32);
      float2 dx = make_float2(0.f, 0.f), dyy = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const int col = 64 * h + 32 * c + 2 * k;
          const float4 wx = lds4(&sv->w0x[col]);
          const float4 wy = lds4(&sv->w0y[col]);
          const float2 g0 = dact_pair(make_float2(v[32 * c + 2 * k], v[32 * c + 2 * k + 1]), m1[c], k);
          const float2 g1 = dact_pair(make_float2(v[32 * c + 2 * k + 2], v[32 * c + 2 * k + 3]), m1[c], k + 1);
          dx = fma2(g0, make_float2(wx.x, wx.y), dx);
          dyy = fma2(g0, make_float2(wy.x, wy.y), dyy);
          dx = fma2(g1, make_float2(wx.z, wx.w), dx);
          dyy = fma2(g1, make_float2(wy.z, wy.w), dyy);
        }
      }
      *reinterpret_cast<float2*>(&sv->xdy[s][r][2 * h]) = make_float2(dx.x + dx.y, dyy.x + dyy.y);
      pair_sync(s, q);  // (the next tile's MMAs follow run_layer's fence + group barrier)
      if (h == 0 && valid) {
        const float4 p = lds4(&sv->xdy[s][r][0]);
        a.dy[row] = make_float2(p.x + p.z, p.y + p.w);
      }
    }
  }
  cta_stamp(a.trace, 0, 2);
  // this CTA's loss partial (fp64), warps in order
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) lacc += __shfl_xor_sync(0xffffffffu, lacc, w);
  if (lane == 0) sv->loss[warp] = lacc;
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < kThreadsF / 32; ++w) sum += sv->loss[w];
    a.loss_part[j] = sum;
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}


// k_dfwd (a7, the forward half of the D step on [X_real; Y_fake], P:93,
// P:146): per 128-row tile, H_1 (SIMT) -> three MMA layers with the
// activations in TMEM (as k_gstep) -> head: z, BCE (labels 1 for rows <
// n_real, else label_rest), dz, G_4 = dz w (.) LeakyReLU'(Z_4).  What the
// per-layer backward passes read goes to HBM in their plane-tile format: the
// hi planes and sign masks of H_2 and H_3 (the wgrad uses the hi plane only,
// R28) and, for G_4 = dz w (.) LeakyReLU'(Z_4), either its planes (bf16) or
// -- fp32-class -- just dz and the sign bits of Z_4 (20 B/row instead of 512:
// the next pass regenerates the planes in shared memory, k_tc_layers.cu
// kGenG); plus the logits, the per-CTA loss and the head gradient partials
// (dW_head = sum dz H_4, db_head = sum dz).
template <bool kSplit, bool kGenOut>
__global__ void __launch_bounds__(kThreadsF, 1) k_dfwd(const __grid_constant__ DFwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  cta_stamp(a.trace, 1, 0);
  constexpr uint32_t TBw = (kSplit ? 2 : 1) * kPlaneF;
  constexpr int64_t TB = (kSplit ? 2 : 1) * (int64_t)kPlaneF;  // HBM plane tile
  SmemVec* sv = reinterpret_cast<SmemVec*>(smem + 3 * TBw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (smem_u32(smem) & 1023u) __trap();
  const uint32_t wbase = smem_u32(smem);
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) mbar_init(&sv->acc_full[s], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&sv->tmem);
  for (int l = 0; l < 3; ++l) stage_w<kSplit>(a.W[l + 1], wbase + l * TBw, wbase + l * TBw + kPlaneF);
  for (int i = tid; i < 128; i += kThreadsF) {
    for (int l = 0; l < 3; ++l) sv->b[l][i] = a.b[l + 1][i];
    sv->w4[i] = a.w4[i];
    sv->aw4[i] = a.alpha * a.w4[i];
    sv->w0x[i] = a.W[0][2 * i];
    sv->w0y[i] = a.W[0][2 * i + 1];
    sv->b0[i] = a.b[0][i];
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sv->tmem;
  cta_stamp(a.trace, 1, 1);
  const int64_t ntiles = (a.rows + 127) / 128;
  const int j = blockIdx.x, n = gridDim.x;
  const int nmine = ntiles > j ? (int)((ntiles - 1 - j) / n + 1) : 0;

  const int s = warp >> 3, w8 = warp & 7, q = w8 & 3, h = w8 >> 2;
  const int r = 32 * q + lane;
  const uint32_t lanes = (uint32_t)(32 * q) << 16;
  const uint32_t slot = tmem + 256u * s;
  const uint32_t accT = slot + lanes + 64u * h;
  const uint32_t ahT = slot + 128u + lanes + 32u * h;
  const uint32_t alT = ahT + 64u;
  const float2 alpha2 = make_float2(a.alpha, a.alpha);
  const float b4 = *a.b4;
  uint32_t acc_ph = 0;
  double lacc = 0.0;
  float gacc0 = 0.f, gacc1 = 0.f, gbacc = 0.f;  // head gradient partials: columns 64 h + lane, 64 h + 32 + lane; dz
  auto put_a = [&](int c, const uint32_t* hw, const uint32_t* lw) {
    tmem_st16(ahT + 16u * c, hw);
    if (kSplit) tmem_st16(alT + 16u * c, lw);
  };
  int cur_i = 0;
  unsigned long long* tr = a.trace ? a.trace + 2 * 64 * 6 * 4 : nullptr;
  auto stamp = [&](int p, int k) {
    if (tr && j == 0 && w8 == 0 && lane == 0 && cur_i / 2 < 64) tr[((s * 64 + cur_i / 2) * 6 + p) * 4 + k] = clock64();
  };
  auto run_layer = [&](int p) {
    stamp(p, 0);
    tmem_st_wait();
    tc_fence_before();
    group_sync(s);
    stamp(p, 1);
    if (w8 == 0) {
      tc_fence_after();
      issue_layer<kSplit>(slot, wbase, p);
      mma_commit_warp(&sv->acc_full[s]);
    }
    stamp(p, 2);
    mbar_wait(&sv->acc_full[s], acc_ph & 1u);
    ++acc_ph;
    tc_fence_after();
    stamp(p, 3);
  };
  auto act_pair = [&](float2 z, int k, uint32_t& hw, uint32_t& lw, uint32_t& m) {
    const float2 tt = mul2(z, alpha2);
    split2(make_float2(fmaxf(z.x, tt.x), fmaxf(z.y, tt.y)), hw, lw);
    m |= pos_bits(hw, k);
  };
  for (int i = s; i < nmine; i += 2) {
    cur_i = i;
    const int64_t t = (int64_t)j + (int64_t)i * n;
    const int64_t row = t * 128 + r;
    const bool valid = row < a.rows;
    const float2 x = valid ? __ldg(a.X + row) : make_float2(0.f, 0.f);
    if (kPrefetchX && w8 == 0 && lane == 0 && i + 2 < nmine) {  // this slot's next tile's rows into L2
      const int64_t r0 = (t + 2 * (int64_t)n) * 128;
      prefetch_rows(a.X, r0, a.rows - r0 < 128 ? a.rows - r0 : 128);
    }
    {  // H_1
      const float2 X0 = make_float2(x.x, x.x), X1 = make_float2(x.y, x.y);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hw[16], lw[16], m = 0u;
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const int col = 64 * h + 32 * c + 2 * k;
          const float4 wx = lds4(&sv->w0x[col]);
          const float4 wy = lds4(&sv->w0y[col]);
          const float4 bb = lds4(&sv->b0[col]);
          act_pair(fma2(X0, make_float2(wx.x, wx.y), fma2(X1, make_float2(wy.x, wy.y), make_float2(bb.x, bb.y))), k,
                   hw[k], lw[k], m);
          act_pair(fma2(X0, make_float2(wx.z, wx.w), fma2(X1, make_float2(wy.z, wy.w), make_float2(bb.z, bb.w))),
                   k + 1, hw[k + 1], lw[k + 1], m);
        }
        put_a(c, hw, lw);
      }
    }
    // W_1, W_2: H_{l+1} -> TMEM A and, hi plane + mask, to HBM (H_2, H_3)
#pragma unroll 1
    for (int l = 0; l < 2; ++l) {
      run_layer(l);
      uint8_t* plane = (l == 0 ? a.h2 : a.h3) + t * TB;
      float v[64];
      tmem_ld32x2(accT, accT + 32u, v, v + 32);
      uint32_t mb[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hw[16], lw[16], m = 0u;
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const float4 bq = lds4(&sv->b[l][64 * h + 32 * c + 2 * k]);
          act_pair(add2(make_float2(v[32 * c + 2 * k], v[32 * c + 2 * k + 1]), make_float2(bq.x, bq.y)), k, hw[k],
                   lw[k], m);
          act_pair(add2(make_float2(v[32 * c + 2 * k + 2], v[32 * c + 2 * k + 3]), make_float2(bq.z, bq.w)), k + 1,
                   hw[k + 1], lw[k + 1], m);
        }
        put_a(c, hw, lw);
        if (!valid) {  // rows past the end are zeros in HBM (the backward reads whole tiles)
#pragma unroll
          for (int k = 0; k < 16; ++k) hw[k] = 0u;
          m = 0u;
        }
        mb[c] = m;
        store_plane_words(plane, r, h, c, hw);
      }
      reinterpret_cast<uint2*>((l == 0 ? a.m2 : a.m3) + t * 128 + r)[h] = make_uint2(mb[0], mb[1]);
    }
    // head.  Pass 1: H_4 = LeakyReLU(Z_4) and its dot with w; H_4 goes back
    // into the accumulator columns for pass 2 (its sign is Z_4's)
    run_layer(2);
    float2 dot = make_float2(0.f, 0.f);
    {
      float v[64];
      tmem_ld32x2(accT, accT + 32u, v, v + 32);
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        const int col = 64 * h + 2 * k;
        const float4 bq = lds4(&sv->b[2][col]);
        const float4 wq = lds4(&sv->w4[col]);
        const float2 z0 = add2(make_float2(v[2 * k], v[2 * k + 1]), make_float2(bq.x, bq.y));
        const float2 z1 = add2(make_float2(v[2 * k + 2], v[2 * k + 3]), make_float2(bq.z, bq.w));
        const float2 t0 = mul2(z0, alpha2), t1 = mul2(z1, alpha2);
        const float2 h0 = make_float2(fmaxf(z0.x, t0.x), fmaxf(z0.y, t0.y));
        const float2 h1 = make_float2(fmaxf(z1.x, t1.x), fmaxf(z1.y, t1.y));
        dot = fma2(h0, make_float2(wq.x, wq.y), dot);
        dot = fma2(h1, make_float2(wq.z, wq.w), dot);
        v[2 * k] = h0.x;
        v[2 * k + 1] = h0.y;
        v[2 * k + 2] = h1.x;
        v[2 * k + 3] = h1.y;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st16(accT + 16u * c, reinterpret_cast<const uint32_t*>(v + 16 * c));
    }
    sv->xdot[s][r][h] = dot.x + dot.y;
    pair_sync(s, q);
    const float zz = (sv->xdot[s][r][0] + sv->xdot[s][r][1]) + b4;
    const float tl = (row < a.n_real) ? 1.f : a.label_rest;
    const float dz = valid ? (sigmoid_f(zz) - tl) * a.scale : 0.f;
    if (valid && h == 0) {
      a.logits[row] = zz;
      lacc += (double)(tl * softplus_neg(zz) + (1.f - tl) * softplus_neg(-zz));
      gbacc += dz;
    }
    uint8_t* gplane = kGenOut ? nullptr : a.g4 + t * TB;
    const float2 dz2 = make_float2(dz, dz);
    if (kGenOut && h == 0) a.dz[row] = dz;  // the backward generates G_4 from dz and the sign bits (kGenG)
    {
      float v[64];
      tmem_st_wait();  // pass 1's H_4 stores
      tmem_ld32x2(accT, accT + 32u, v, v + 32);
      uint32_t mb[2] = {0u, 0u};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hw[16], lw[16];
        float g[32];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const int col = 64 * h + 32 * c + 2 * k;
          const float4 wq = lds4(&sv->w4[col]);
          const float4 aq = lds4(&sv->aw4[col]);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float2 z = make_float2(v[32 * c + 2 * (k + u)], v[32 * c + 2 * (k + u) + 1]);  // H_4 (sign of Z_4)
            const float2 hd = mul2(dz2, z);  // dz H_4
            g[2 * (k + u)] = hd.x;
            g[2 * (k + u) + 1] = hd.y;
            if (!kGenOut) {
              const float2 w = u ? make_float2(wq.z, wq.w) : make_float2(wq.x, wq.y);
              const float2 wa = u ? make_float2(aq.z, aq.w) : make_float2(aq.x, aq.y);
              split2(mul2(dz2, make_float2(z.x > 0.f ? w.x : wa.x, z.y > 0.f ? w.y : wa.y)), hw[k + u], lw[k + u]);
            } else {  // sign bits of Z_4, column 2kk -> bit kk, 2kk + 1 -> bit 16 + kk
              mb[c] |= (z.x > 0.f ? 1u : 0u) << (k + u);
              mb[c] |= (z.y > 0.f ? 1u : 0u) << (16 + k + u);
            }
          }
        }
        if (!kGenOut) {
          store_plane_words(gplane, r, h, c, hw);
          if (kSplit) store_plane_words(gplane + kPlaneF, r, h, c, lw);
        }
        const float cs = colsum32(g, lane);
        if (c == 0) gacc0 += cs;
        else gacc1 += cs;
      }
      if (kGenOut) reinterpret_cast<uint2*>(a.m4 + t * 128 + r)[h] = make_uint2(valid ? mb[0] : 0u, valid ? mb[1] : 0u);
    }
    tc_fence_before();  // this tile's accumulator reads precede the next tile's MMAs
    stamp(3, 0);
    stamp(3, 1);
    stamp(3, 2);
    stamp(3, 3);
  }
  cta_stamp(a.trace, 1, 2);
  // per-CTA partials in a fixed order: head gradient [128] + bias, loss (fp64)
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    lacc += __shfl_xor_sync(0xffffffffu, lacc, w);
    gbacc += __shfl_xor_sync(0xffffffffu, gbacc, w);
  }
  float* sred = sv->red;  // [16 warps][64 + 1]
  tc_fence_before();
  __syncthreads();
  sred[warp * 65 + lane] = gacc0;
  sred[warp * 65 + 32 + lane] = gacc1;
  if (lane == 0) {
    sred[warp * 65 + 64] = gbacc;
    sv->loss[warp] = lacc;
  }
  __syncthreads();
  if (tid < 129) {
    float v = 0.f;
    if (tid < 128) {
      const int hh = tid >> 6, cc = tid & 63;
      for (int ss = 0; ss < 2; ++ss)
        for (int qq = 0; qq < 4; ++qq) v += sred[(8 * ss + 4 * hh + qq) * 65 + cc];
    } else {
      for (int w = 0; w < 16; ++w) v += sred[w * 65 + 64];
    }
    a.part_head[(int64_t)j * 129 + tid] = v;
  }
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < kThreadsF / 32; ++w) sum += sv->loss[w];
    a.loss_part[j] = sum;
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

static unsigned long long* g_ftrace = nullptr;
unsigned long long* fused_trace_buffer() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SAGIPS_FUSED_TRACE");
    on = (e && e[0] == '1') ? 1 : 0;
    if (on) {
      cudaMalloc(&g_ftrace, sizeof(unsigned long long) * (kFTracePhaseWords + 2 * 256 * 4));
      cudaMemset(g_ftrace, 0, sizeof(unsigned long long) * (kFTracePhaseWords + 2 * 256 * 4));
    }
  }
  return g_ftrace;
}
void fused_trace_report() {
  if (!g_ftrace) return;
  std::vector<unsigned long long> h(kFTracePhaseWords + 2 * 256 * 4);
  cudaDeviceSynchronize();
  cudaMemcpy(h.data(), g_ftrace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
  // per phase: epilogue (previous accumulator ready -> this warp done), waiting
  // for the group, MMA issue, MMA completion wait; cycles, mean over tiles 1..
  for (int kern = 0; kern < 2; ++kern) {
    const int np = kern == 0 ? 6 : 4;
    const unsigned long long* H = h.data() + (size_t)kern * 2 * 64 * 6 * 4;
    double acc[6][4] = {};
    int cnt[6] = {};
    for (int s = 0; s < 2; ++s)
      for (int t = 1; t < 64; ++t)
        for (int p = 0; p < np; ++p) {
          const unsigned long long* e = &H[((s * 64 + t) * 6 + p) * 4];
          if (!e[0] || !e[3]) continue;
          const unsigned long long prev =
              p > 0 ? H[((s * 64 + t) * 6 + p - 1) * 4 + 3] : H[((s * 64 + t - 1) * 6 + np - 1) * 4 + 3];
          if (!prev || prev > e[0]) continue;
          acc[p][0] += (double)(e[0] - prev);
          acc[p][1] += (double)(e[1] - e[0]);
          acc[p][2] += (double)(e[2] - e[1]);
          acc[p][3] += (double)(e[3] - e[2]);
          cnt[p]++;
        }
    fprintf(stderr, "sagips fused trace %s (CTA 0, cycles per phase: epilogue | group wait | MMA issue | MMA wait)\n",
            kern == 0 ? "k_gstep" : "k_dfwd");
    for (int p = 0; p < np; ++p)
      if (cnt[p])
        fprintf(stderr, "  phase %d: %7.0f | %6.0f | %6.0f | %6.0f  (%d samples)\n", p, acc[p][0] / cnt[p],
                acc[p][1] / cnt[p], acc[p][2] / cnt[p], acc[p][3] / cnt[p], cnt[p]);
    // per-CTA timeline of the last traced launch: prologue, tile loop end spread
    const unsigned long long* C = h.data() + kFTracePhaseWords + (size_t)kern * 256 * 4;
    std::vector<double> pro, loop_end;
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < 256; ++c)
      if (C[c * 4] && C[c * 4] < t0) t0 = C[c * 4];
    int slowest = -1;
    double worst = 0;
    for (int c = 0; c < 256; ++c) {
      if (!C[c * 4] || !C[c * 4 + 2]) continue;
      pro.push_back((double)(C[c * 4 + 1] - C[c * 4]) * 1e-3);
      const double e = (double)(C[c * 4 + 2] - t0) * 1e-3;
      loop_end.push_back(e);
      if (e > worst) { worst = e; slowest = (int)C[c * 4 + 3]; }
    }
    if (!loop_end.empty()) {
      std::sort(pro.begin(), pro.end());
      std::sort(loop_end.begin(), loop_end.end());
      const size_t n = loop_end.size();
      fprintf(stderr, "  %zu CTAs: prologue %.2f us (median), tile loop done at %.1f / %.1f / %.1f us (min / median / max; slowest on SM %d)\n",
              n, pro[n / 2], loop_end[0], loop_end[n / 2], loop_end[n - 1], slowest);
    }
  }
}

static int sm_count_f() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static size_t gstep_smem(bool split) { return 3 * (split ? 2 : 1) * kPlaneF + sizeof(SmemVec) + 1024; }

int fused_grid(int64_t rows) {
  return (int)std::min<int64_t>(std::max<int64_t>((rows + 127) / 128, 1), sm_count_f());
}

void launch_dfwd(bool split, const DFwdArgs& a, cudaStream_t st) {
  static bool configured[4] = {false, false, false, false};
  const size_t smem = gstep_smem(split);
  const bool gen = a.g4 == nullptr;  // G_4 as dz + sign bits (the next pass regenerates it)
  auto kern = split ? (gen ? k_dfwd<true, true> : k_dfwd<true, false>) : (gen ? k_dfwd<false, true> : k_dfwd<false, false>);
  const int ci = 2 * (split ? 1 : 0) + (gen ? 1 : 0);
  if (!configured[ci]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[ci] = true;
  }
  kern<<<fused_grid(a.rows), kThreadsF, smem, st>>>(a);
  count_launch();
}

void launch_gstep(bool split, const GStepArgs& a, cudaStream_t st) {
  static bool configured[2] = {false, false};
  const size_t smem = gstep_smem(split);
  auto kern = split ? k_gstep<true> : k_gstep<false>;
  if (!configured[split]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[split] = true;
  }
  kern<<<fused_grid(a.rows), kThreadsF, smem, st>>>(a);
  count_launch();
}

}  // namespace sagips
