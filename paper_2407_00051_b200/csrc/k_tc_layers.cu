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
#include <cstdlib>

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

struct Params0 {  // layer-0 parameters, column-contiguous
  float w0x[128];
  float w0y[128];
  float b0[128];
};

__device__ __forceinline__ float lrelu(float z, float a) { return z > 0.f ? z : z * a; }

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

// hi = bf16(a,b), lo = bf16(a - hi, b - hi)
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

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

// SIMT producer of H_1 planes for one tile (warps 0-3, warp w: rows 32w..32w+31;
// lane l: columns 4l..4l+3).  xr = this lane's prefetched input row 32w + l.
template <bool kSplit>
__device__ __forceinline__ void produce_h1(float2 xr, bool xvalid, const Params0* p0, float alpha, uint32_t hi,
                                           uint32_t lo, int w, int l) {
  const float4 wx = *reinterpret_cast<const float4*>(&p0->w0x[4 * l]);
  const float4 wy = *reinterpret_cast<const float4*>(&p0->w0y[4 * l]);
  const float4 bb = *reinterpret_cast<const float4*>(&p0->b0[4 * l]);
  const unsigned vbits = __ballot_sync(0xffffffffu, xvalid);
  const uint32_t cbase = (uint32_t)(l >> 4) * 16384u + 8u * (uint32_t)(l & 1);
  const int jj = (l >> 1) & 7;
#pragma unroll 1
  for (int i0 = 0; i0 < 32; i0 += 4) {
    uint32_t hw[4][2], lw[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // 4 independent rows in flight
      const float x0 = __shfl_sync(0xffffffffu, xr.x, i0 + u), x1 = __shfl_sync(0xffffffffu, xr.y, i0 + u);
      // branch-free: rows past the end are multiplied by 0 (their x is 0, so the values are finite)
      const float ok = ((vbits >> (i0 + u)) & 1u) ? 1.f : 0.f;
      const float a = ok * lrelu(fmaf(x0, wx.x, fmaf(x1, wy.x, bb.x)), alpha);
      const float b = ok * lrelu(fmaf(x0, wx.y, fmaf(x1, wy.y, bb.y)), alpha);
      const float c = ok * lrelu(fmaf(x0, wx.z, fmaf(x1, wy.z, bb.z)), alpha);
      const float d = ok * lrelu(fmaf(x0, wx.w, fmaf(x1, wy.w, bb.w)), alpha);
      split2(a, b, hw[u][0], lw[u][0]);
      split2(c, d, hw[u][1], lw[u][1]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = 32 * w + i0 + u;
      const uint32_t off = cbase + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 128u + ((uint32_t)(jj ^ (r & 7)) << 4);
      sts64(hi + off, hw[u][0], hw[u][1]);
      if (kSplit) sts64(lo + off, lw[u][0], lw[u][1]);
    }
  }
}

// ---- optional timeline trace (SAGIPS_TRACE=1): globaltimer stamps per tile
// for CTAs 0..3: 0 operands staged, 1 MMA started, 2 epilogue got the
// accumulator, 3 epilogue released it.
constexpr int kTraceLaunches = 32, kTraceCtas = 4, kTraceTiles = 256;
__device__ __forceinline__ void trace_pt(unsigned long long* tr, int i, int k) {
  if (tr && blockIdx.x < kTraceCtas && i < kTraceTiles) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[((size_t)blockIdx.x * kTraceTiles + i) * 4 + k] = t;
  }
}

__device__ __forceinline__ void check_smem_alignment(const void* p) {
  if (smem_u32(p) & 1023u) __trap();  // SW128 operands need 1024-byte alignment
}

}  // namespace

// ============================================================== forward
struct FwdArgs {
  const uint8_t* A;     // input plane tiles (mid, head)
  const float* X;       // [rows][2] (first)
  const float* W0;      // [128][2] (first)
  const float* b0;      // [128] (first)
  const float* W;       // [128][128] this layer
  const float* bias;    // [128]
  uint8_t* C;           // output plane tiles (mid, first: H; head: G)
  uint4* mask;          // [tiles*128] sign masks of H (mid, first)
  int64_t rows;
  float alpha;
  // head
  const float* w_head;  // [128]
  const float* b_head;  // [1]
  int64_t n_real;       // rows < n_real carry label 1, the rest label_rest
  float label_rest;
  float scale;          // 1/(number of rows in the mean)
  float* logits;        // [rows]
  float* part_head;     // [grid*4][129]: sum dz*H (128), sum dz
  double* loss_part;    // [grid]
  int want_wgrad;
  unsigned long long* trace;
};

template <bool kSplit, bool kFirst, bool kHead>
__global__ void __launch_bounds__(kThreads, 1) k_fwd(FwdArgs a) {
  constexpr int P = kSplit ? 2 : 1;
  constexpr uint32_t TB = P * kPlane;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sW = smem;
  uint8_t* sA = sW + TB;          // 2 stages
  uint8_t* sStg = sA + 2 * TB;    // 8 x 4 KiB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + kEW * kStg);
  uint64_t* full = bars;          // [2]
  uint64_t* empty = bars + 2;     // [2]
  uint64_t* tfull = bars + 4;     // [2]
  uint64_t* tempty = bars + 6;    // [2]
  double* sloss = reinterpret_cast<double*>(bars + 8);  // [8]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sloss + 8);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);  // [128]
  float* swh = sbias + 128;                                 // [128] (head)
  float* pdot = swh + 128;                                  // [2 halves][128] (head)
  Params0* p0 = reinterpret_cast<Params0*>(swh);            // (first; aliases swh + pdot)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    check_smem_alignment(smem);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], kFirst ? 32 * kPW : 1);
      mbar_init(&empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEW);
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
  if (warp < kPW) stage_weights<kSplit>(a.W, smem_u32(sW), smem_u32(sW + kPlane), warp, lane);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto tile_of = [&](int i) { return blockIdx.x + (int64_t)i * gridDim.x; };

  if (warp < kPW) {
    // ---------------- SIMT producers of H_1 (first layer only)
    if (kFirst) {
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
      for (int i = 0; i < nmine; ++i) {
        const int s = i & 1;
        bool ok_next;
        const float2 xn = load_x(i + 1, ok_next);
        mbar_wait(&empty[s], ((i >> 1) & 1) ^ 1);
        const uint32_t st = smem_u32(sA + s * TB);
        produce_h1<kSplit>(xr, ok, p0, a.alpha, st, st + kPlane, warp, lane);
        fence_proxy_async_smem();
        mbar_arrive(&full[s]);
        if (warp == 0 && lane == 0) trace_pt(a.trace, i, 0);
        xr = xn;
        ok = ok_next;
      }
    }
  } else if (warp == kLoadWarp) {
    // ---------------- bulk loader
    if (!kFirst && lane == 0) {
      for (int i = 0; i < nmine; ++i) {
        const int s = i & 1;
        if (i + 1 < nmine) prefetch_l2(a.A + tile_of(i + 1) * TB, TB);
        mbar_wait(&empty[s], ((i >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], TB);
        bulk_g2s(smem_u32(sA + s * TB), a.A + tile_of(i) * TB, TB, &full[s]);
        trace_pt(a.trace, i, 0);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
      const uint32_t bh = smem_u32(sW), bl = bh + kPlane;
      for (int i = 0; i < nmine; ++i) {
        const int s = i & 1, b = i & 1;
        mbar_wait(&full[s], (i >> 1) & 1);
        mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        trace_pt(a.trace, i, 1);
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
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warp e -> TMEM lane quarter q, column half h
    const int e = warp - kPW;
    const int q = warp & 3;
    const int h = e >> 2;
    const int cb = 64 * h;
    const uint32_t stg = smem_u32(sStg) + e * kStg;
    float gacc[2] = {0.f, 0.f};   // head: sum dz*H, columns cb + 32c + lane
    float gbacc = 0.f;
    double lacc = 0.0;
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = tile_of(i);
      const int b = i & 1;
      const int64_t row = t * 128 + 32 * q + lane;
      const bool valid = row < a.rows;
      uint8_t* dst = a.C + t * TB + h * 16384 + q * 4096;
      mbar_wait(&tfull[b], (i >> 1) & 1);
      if (e == 0 && lane == 0) trace_pt(a.trace, i, 2);
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * 128 + cb) + ((uint32_t)(32 * q) << 16);
      uint32_t lo[32];
      stage_free(lane);
      if (!kHead) {
        uint32_t mb[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
          uint32_t m = 0;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float z = v[k] + sbias[cb + 32 * c + k];
            m |= (z > 0.f ? 1u : 0u) << k;
            v[k] = valid ? lrelu(z, a.alpha) : 0.f;
          }
          mb[c] = valid ? m : 0u;
          uint32_t hw[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) split2(v[2 * k], v[2 * k + 1], hw[k], lo[16 * c + k]);
          stage_words(stg, lane, c, hw);
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        if (e == 0 && lane == 0) trace_pt(a.trace, i, 3);
        flush_stage(stg, dst, lane);
        reinterpret_cast<uint2*>(a.mask + t * 128 + 32 * q + lane)[h] = make_uint2(mb[0], mb[1]);
      } else {
        // pass 1: partial z = H . w over this warp's 64 columns
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int cc = cb + 32 * c + k;
            dot = fmaf(lrelu(v[k] + sbias[cc], a.alpha), swh[cc], dot);
          }
        }
        epi_sync();  // previous tile's reads of pdot done
        pdot[h * 128 + 32 * q + lane] = dot;
        epi_sync();
        const float z = pdot[32 * q + lane] + pdot[128 + 32 * q + lane] + *a.b_head;
        const float tl = (row < a.n_real) ? 1.f : a.label_rest;
        const float dz = valid ? (sigmoid_f(z) - tl) * a.scale : 0.f;
        if (valid && h == 0) {
          a.logits[row] = z;
          lacc += (double)(tl * softplus_neg(z) + (1.f - tl) * softplus_neg(-z));
          gbacc += dz;
        }
        // pass 2: G = dz * w * LeakyReLU'(Z) -> planes; head gradient dz * H
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
          float g[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int cc = cb + 32 * c + k;
            const float zz = v[k] + sbias[cc];
            g[k] = dz * lrelu(zz, a.alpha);
            v[k] = dz * swh[cc] * (zz > 0.f ? 1.f : a.alpha);
          }
          uint32_t hw[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) split2(v[2 * k], v[2 * k + 1], hw[k], lo[16 * c + k]);
          stage_words(stg, lane, c, hw);
          if (a.want_wgrad) gacc[c] += colsum32(g, lane);
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        if (e == 0 && lane == 0) trace_pt(a.trace, i, 3);
        flush_stage(stg, dst, lane);
      }
      if (kSplit) {
        stage_free(lane);
        stage_words(stg, lane, 0, lo);
        stage_words(stg, lane, 1, lo + 16);
        flush_stage(stg, dst + kPlane, lane);
      }
    }
    if (lane == 0) bulk_wait0();
    if (kHead) {
      // per-(CTA, lane quarter) partials; loss per CTA in fp64, fixed order
      const int64_t pq = (int64_t)blockIdx.x * 4 + q;
      if (a.want_wgrad) {
#pragma unroll
        for (int c = 0; c < 2; ++c) a.part_head[pq * 129 + cb + 32 * c + lane] = gacc[c];
      }
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
        gbacc += __shfl_xor_sync(0xffffffffu, gbacc, w);
        lacc += __shfl_xor_sync(0xffffffffu, lacc, w);
      }
      if (lane == 0) {
        if (a.want_wgrad && h == 0) a.part_head[pq * 129 + 128] = gbacc;
        sloss[e] = lacc;
      }
      epi_sync();
      if (e == 0 && lane == 0) {
        double s = 0.0;
        for (int j = 0; j < kEW; ++j) s += sloss[j];
        a.loss_part[blockIdx.x] = s;
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
  const uint8_t* G;     // G_{l+1} plane tiles
  const uint8_t* H;     // H_l plane tiles (wgrad, not first)
  const uint4* mask;    // sign mask of H_l (not first)
  const float* X;       // [rows][2] (first)
  const float* W0;      // [128][2] (first)
  const float* b0;      // [128] (first)
  const float* W;       // [128][128] W_l
  int64_t rows;
  float alpha;
  uint8_t* Gout;        // G_l plane tiles (not first)
  float* dy;            // [rows][2] (first, no wgrad)
  float* part;          // [grid][128][128] dW_l partials (wgrad)
  float* part_db;       // [grid][128] db_l partials (wgrad)
  float* part_l0;       // [grid*4][384] dW_0 (256, row-major) + db_0 (128) (first, wgrad)
  unsigned long long* trace;
};

template <bool kSplit, bool kFirst, bool kWgrad>
__global__ void __launch_bounds__(kThreads, 1) k_bwd(BwdArgs a) {
  constexpr int P = kSplit ? 2 : 1;
  constexpr uint32_t TB = P * kPlane;
  constexpr bool kDy = kFirst && !kWgrad;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sW = smem;
  uint8_t* sG = sW + TB;     // G stage 0
  uint8_t* sH = sG + TB;     // H stage (wgrad) or G stage 1
  uint8_t* sStg = sH + TB;   // 8 x 4 KiB (dy: the partial-dot exchange)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + kEW * kStg);
  uint64_t* fullG = bars;       // [2]
  uint64_t* emptyG = bars + 2;  // [2]
  uint64_t* fullH = bars + 4;   // [1]
  uint64_t* emptyH = bars + 5;  // [1]
  uint64_t* tfull = bars + 6;   // [2]
  uint64_t* tempty = bars + 8;  // [2]
  uint64_t* wdone = bars + 10;  // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  uint32_t* sOnes = tmem_slot + 4;                           // 512 B of bf16 1.0 (db MMA operand)
  Params0* p0 = reinterpret_cast<Params0*>(sOnes + 128);    // (first)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    check_smem_alignment(smem);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&fullG[i], 1);
      mbar_init(&emptyG[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEW);
    }
    mbar_init(&fullH[0], kFirst ? 32 * kPW : 1);
    mbar_init(&emptyH[0], 1);
    mbar_init(&wdone[0], 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  for (int i = tid; i < 128; i += kThreads) sOnes[i] = 0x3F803F80u;
  if (kFirst) {
    for (int i = tid; i < 128; i += kThreads) {
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
  const uint32_t acc_w = tmem + 256, acc_b = tmem + 384;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto tile_of = [&](int i) { return blockIdx.x + (int64_t)i * gridDim.x; };
  // G stage of tile i: wgrad -> single stage; else a ring of 2 (sG, sH)
  auto g_stage = [&](int i) -> uint8_t* { return (!kWgrad && (i & 1)) ? sH : sG; };

  if (warp < kPW) {
    // ---------------- SIMT producers of H_1 planes (first layer, wgrad)
    if (kFirst && kWgrad) {
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
      const uint32_t hh = smem_u32(sH);
      for (int i = 0; i < nmine; ++i) {
        bool ok_next;
        const float2 xn = load_x(i + 1, ok_next);
        mbar_wait(&emptyH[0], (i & 1) ^ 1);
        produce_h1<kSplit>(xr, ok, p0, a.alpha, hh, hh + kPlane, warp, lane);
        fence_proxy_async_smem();
        mbar_arrive(&fullH[0]);
        xr = xn;
        ok = ok_next;
      }
    }
  } else if (warp == kLoadWarp) {
    // ---------------- bulk loader
    if (lane == 0) {
      for (int i = 0; i < nmine; ++i) {
        const int64_t t = tile_of(i);
        if (i + 1 < nmine) {
          prefetch_l2(a.G + tile_of(i + 1) * TB, TB);
          if (kWgrad && !kFirst) prefetch_l2(a.H + tile_of(i + 1) * TB, TB);
        }
        if (kWgrad && !kFirst) {
          mbar_wait(&emptyH[0], (i & 1) ^ 1);
          mbar_arrive_expect_tx(&fullH[0], TB);
          bulk_g2s(smem_u32(sH), a.H + t * TB, TB, &fullH[0]);
        }
        const int s = kWgrad ? 0 : (i & 1);
        const uint32_t ph = kWgrad ? ((i & 1) ^ 1) : (((i >> 1) & 1) ^ 1);
        mbar_wait(&emptyG[s], ph);
        mbar_arrive_expect_tx(&fullG[s], TB);
        bulk_g2s(smem_u32(g_stage(i)), a.G + t * TB, TB, &fullG[s]);
        trace_pt(a.trace, i, 0);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_d = make_idesc_bf16(128, 128, 0, 1);  // A = G (K-major), B = W (MN-major)
      constexpr uint32_t id_w = make_idesc_bf16(128, 128, 1, 1);  // A = G^T, B = H (both MN-major)
      constexpr uint32_t id_b = make_idesc_bf16(128, 16, 1, 0);   // A = G^T, B = ones (K-major)
      const uint64_t ones = make_desc(smem_u32(sOnes), 128, 256, 0);  // no swizzle: any layout reads 1.0
      const uint32_t wh = smem_u32(sW), wl = wh + kPlane;
      const uint32_t hh = smem_u32(sH), hl = hh + kPlane;
      for (int i = 0; i < nmine; ++i) {
        const int b = i & 1;
        const int s = kWgrad ? 0 : (i & 1);
        mbar_wait(&fullG[s], kWgrad ? (i & 1) : ((i >> 1) & 1));
        const uint32_t zh = smem_u32(g_stage(i)), zl = zh + kPlane;
        if (kWgrad) {
          mbar_wait(&fullH[0], i & 1);
          trace_pt(a.trace, i, 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t km = k * 2048;  // MN-major step (16 rows)
            const uint32_t acc0 = (i > 0 || k > 0) ? 1u : 0u;
            const uint64_t gh = make_desc(zh + km, 16384, 1024), gl = make_desc(zl + km, 16384, 1024);
            mma_step<kSplit>(acc_w, gh, gl, make_desc(hh + km, 16384, 1024), make_desc(hl + km, 16384, 1024), id_w,
                             acc0);
            mma_bf16(acc_b, gh, ones, id_b, acc0);
            if (kSplit) mma_bf16(acc_b, gl, ones, id_b, 1);
          }
          mma_commit(&emptyH[0]);
        }
        mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        if (!kWgrad) trace_pt(a.trace, i, 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32;  // K-major step (16 columns)
          const uint32_t km = k * 2048;
          // dgrad: D[rows][in] = G[rows][out] * W[out][in]
          mma_step<kSplit>(d, make_desc(zh + kk, 16, 1024), make_desc(zl + kk, 16, 1024),
                           make_desc(wh + km, 16384, 1024), make_desc(wl + km, 16384, 1024), id_d, k > 0);
        }
        mma_commit(&emptyG[s]);
        mma_commit(&tfull[b]);
      }
      mma_commit(&wdone[0]);
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
    for (int i = 0; i < nmine; ++i) {
      const int64_t t = tile_of(i);
      const int b = i & 1;
      const int64_t row = t * 128 + 32 * q + lane;
      const bool valid = row < a.rows;
      uint2 mk = make_uint2(0u, 0u);
      float2 x = make_float2(0.f, 0.f);
      if (kFirst) {
        if (valid) x = __ldg(X2 + row);
      } else {
        mk = __ldg(reinterpret_cast<const uint2*>(a.mask + row) + h);
      }
      mbar_wait(&tfull[b], (i >> 1) & 1);
      if (e == 0 && lane == 0) trace_pt(a.trace, i, 2);
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * 128 + cb) + ((uint32_t)(32 * q) << 16);
      if (!kFirst) {
        uint8_t* dst = a.Gout + t * TB + h * 16384 + q * 4096;
        uint32_t lo[32];
        stage_free(lane);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
          const uint32_t m = c ? mk.y : mk.x;
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = valid ? v[k] * (((m >> k) & 1u) ? 1.f : a.alpha) : 0.f;
          uint32_t hw[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) split2(v[2 * k], v[2 * k + 1], hw[k], lo[16 * c + k]);
          stage_words(stg, lane, c, hw);
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        if (e == 0 && lane == 0) trace_pt(a.trace, i, 3);
        flush_stage(stg, dst, lane);
        if (kSplit) {
          stage_free(lane);
          stage_words(stg, lane, 0, lo);
          stage_words(stg, lane, 1, lo + 16);
          flush_stage(stg, dst + kPlane, lane);
        }
      } else {
        // G_1 = acc * LeakyReLU'(Z_1), Z_1 = x W_0^T + b_0 recomputed exactly as the producers do
        float d0 = 0.f, d1 = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(acc + 32 * c, v);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int cc = cb + 32 * c + k;
            const float z1 = fmaf(x.x, p0->w0x[cc], fmaf(x.y, p0->w0y[cc], p0->b0[cc]));
            v[k] = valid ? v[k] * (z1 > 0.f ? 1.f : a.alpha) : 0.f;
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
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const int cc = cb + 32 * c + k;
              d0 = fmaf(v[k], p0->w0x[cc], d0);
              d1 = fmaf(v[k], p0->w0y[cc], d1);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[b]);
        if (e == 0 && lane == 0) trace_pt(a.trace, i, 3);
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
    const int64_t pq = (int64_t)blockIdx.x * 4 + q;
    if (kWgrad && kFirst) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int cc = cb + 32 * c + lane;
        a.part_l0[pq * 384 + 2 * cc] = s0[c];
        a.part_l0[pq * 384 + 2 * cc + 1] = s1[c];
        a.part_l0[pq * 384 + 256 + cc] = sb[c];
      }
    }
    if (kWgrad) {
      // TMEM lane = output feature o, columns = input features; warp (q, h)
      // writes rows 32q.., columns 64h..64h+63 of this CTA's partial
      const int o = 32 * q + lane;
      float* dst = a.part + (int64_t)blockIdx.x * 128 * 128 + (int64_t)o * 128;
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
        a.part_db[(int64_t)blockIdx.x * 128 + o] = nmine > 0 ? v[0] : 0.f;
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
  return 3 * TB + kEW * kStg + 8 * 8 + 8 * 8 + 16 + 4 * (128 + 128 + 256);  // bias, w_head, pdot / Params0
}
static size_t bwd_smem(bool split) {
  const size_t TB = (split ? 2 : 1) * (size_t)kPlane;
  return 3 * TB + kEW * kStg + 12 * 8 + 16 + 512 + sizeof(Params0);
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
size_t plane_tile_bytes(bool split) { return (split ? 2 : 1) * (size_t)kPlane; }

void launch_tc_fwd(bool split, int kind, const FwdLaunch& L, cudaStream_t st) {
  configure_layers();
  FwdArgs a{};
  a.A = L.A; a.X = L.X; a.W0 = L.W0; a.b0 = L.b0; a.W = L.W; a.bias = L.bias; a.C = L.C; a.mask = L.mask;
  a.rows = L.rows; a.alpha = L.alpha; a.w_head = L.w_head; a.b_head = L.b_head; a.n_real = L.n_real;
  a.label_rest = L.label_rest; a.scale = L.scale; a.logits = L.logits; a.part_head = L.part_head;
  a.loss_part = L.loss_part; a.want_wgrad = L.want_wgrad;
  a.trace = trace_slot();
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = fwd_smem(split);
  if (split) {
    if (kind == FWD_FIRST) k_fwd<true, true, false><<<grid, kThreads, sm, st>>>(a);
    else if (kind == FWD_MID) k_fwd<true, false, false><<<grid, kThreads, sm, st>>>(a);
    else k_fwd<true, false, true><<<grid, kThreads, sm, st>>>(a);
  } else {
    if (kind == FWD_FIRST) k_fwd<false, true, false><<<grid, kThreads, sm, st>>>(a);
    else if (kind == FWD_MID) k_fwd<false, false, false><<<grid, kThreads, sm, st>>>(a);
    else k_fwd<false, false, true><<<grid, kThreads, sm, st>>>(a);
  }
  count_launch();
}

void launch_tc_bwd(bool split, bool first, bool wgrad, const BwdLaunch& L, cudaStream_t st) {
  configure_layers();
  BwdArgs a{};
  a.G = L.G; a.H = L.H; a.mask = L.mask; a.X = L.X; a.W0 = L.W0; a.b0 = L.b0; a.W = L.W; a.rows = L.rows;
  a.alpha = L.alpha; a.Gout = L.Gout; a.dy = L.dy; a.part = L.part; a.part_db = L.part_db; a.part_l0 = L.part_l0;
  a.trace = trace_slot();
  const int grid = tc_layers_grid(L.rows);
  const size_t sm = bwd_smem(split);
#define SAGIPS_BWD_LAUNCH(S)                                                                   \
  if (!first && wgrad) k_bwd<S, false, true><<<grid, kThreads, sm, st>>>(a);                   \
  else if (first && wgrad) k_bwd<S, true, true><<<grid, kThreads, sm, st>>>(a);                \
  else if (!first) k_bwd<S, false, false><<<grid, kThreads, sm, st>>>(a);                      \
  else k_bwd<S, true, false><<<grid, kThreads, sm, st>>>(a);
  if (split) {
    SAGIPS_BWD_LAUNCH(true)
  } else {
    SAGIPS_BWD_LAUNCH(false)
  }
#undef SAGIPS_BWD_LAUNCH
  count_launch();
}

void launch_sum_parts(const float* part, int nparts, int64_t ld, int n, float* out, cudaStream_t st) {
  k_sum_parts<<<(n + 31) / 32, 256, 0, st>>>(part, nparts, ld, n, out);
  count_launch();
}

}  // namespace sagips
