// k_tc_gemm.cu -- discriminator hidden layers (128 -> 128) on the
// 5th-generation tensor cores: tcgen05.mma (kind::f16, bf16 operands, fp32
// accumulation in TMEM), operands staged in 128-byte-swizzled shared memory,
// accumulators read back with tcgen05.ld for fused epilogues.
//
// Two operand modes:
//   bf16   : one MMA per K step                         (SAGIPS_PREC_BF16)
//   bf16x3 : x = hi + lo (two bf16), A*B ~ hi*hi + hi*lo + lo*hi, three MMAs
//            per K step -- fp32-class accuracy (loss 2e-7, grads 6e-4 in the
//            DESIGN.md emulation), used for SAGIPS_PREC_FP32.
//
// k_tc_rows : one 128-row tile per iteration, persistent over tiles;
//             C[rows][128] = epi(A[rows][128] * op(W)), op(W) = W^T (forward,
//             B K-major) or W (dgrad, B MN-major); epilogues bias+LeakyReLU
//             or "times LeakyReLU'(H_prev)".  MMA of tile i overlaps the
//             epilogue of tile i-1 (double-buffered smem and TMEM).
// k_tc_wgrad: split-K over rows: dW[128 out][128 in] += dZ^T H per 64/128-row
//             block (both operands MN-major views of row-major tiles), and
//             db = dZ^T 1 with an N=16 MMA against a ones tile; one fp32
//             partial per CTA, summed in a fixed order afterwards.
#include "ctx.h"
#include "tc_util.cuh"

namespace sagips {

using namespace tc;

constexpr int kTcThreads = 256;
constexpr uint32_t kTile = 128 * 128 * 2;  // bytes of one [128][128] bf16 SW128 tile

// [R][128] fp32 rows [r0, r0+R) of a row-major matrix -> SW128 bf16 tile(s)
template <bool kSplit, int R>
__device__ __forceinline__ void stage_rows(const float* __restrict__ g, int64_t ld, int64_t r0, int64_t nrows,
                                           uint8_t* s_hi, uint8_t* s_lo) {
  for (int q = threadIdx.x; q < R * 16; q += blockDim.x) {
    const int r = q >> 4, j = q & 15;
    const int64_t gr = r0 + r;
    float x[8];
    if (gr < nrows) {
      const float4* p = reinterpret_cast<const float4*>(g + gr * ld + 8 * j);
      const float4 a = __ldg(p), b = __ldg(p + 1);
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = 0.f;
    }
    const uint32_t off = sw128_chunk(r, j, R);
    if (kSplit) {
      uint4 hi, lo;
      split_bf16(x, hi, lo);
      *reinterpret_cast<uint4*>(s_hi + off) = hi;
      *reinterpret_cast<uint4*>(s_lo + off) = lo;
    } else {
      *reinterpret_cast<uint4*>(s_hi + off) =
          make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
    }
  }
}

struct RowsArgs {
  const float* A;      // [rows][128]
  const float* W;      // [128][128] (W_l[out][in])
  float* C;            // [rows][128]
  int64_t rows;
  const float* bias;   // EPI_BIAS_ACT
  const float* Hprev;  // EPI_ACT_GRAD: [rows][128]
  float alpha;
  int epi;
};

template <bool kSplit, bool kDgrad>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_rows(RowsArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int P = kSplit ? 2 : 1;             // operand planes (hi[, lo])
  uint8_t* sW = base;                            // P tiles
  uint8_t* sA = base + P * kTile;                // 2 stages x P tiles
  uint64_t* bar = reinterpret_cast<uint64_t*>(sA + 2 * P * kTile);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  if (a.epi == EPI_BIAS_ACT && tid < 128) sbias[tid] = a.bias[tid];
  stage_rows<kSplit, 128>(a.W, 128, 0, 128, sW, sW + kTile);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t ntiles = (a.rows + 127) / 128;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  constexpr uint32_t idesc = make_idesc_bf16(128, 128, 0, kDgrad ? 1 : 0);

  auto epilogue = [&](int j) {
    const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
    mbar_wait(&bar[j & 1], (j >> 1) & 1);
    tc_fence_after();
    const int lb = 32 * (warp & 3);
    const int col0 = 64 * (warp >> 2);
    const int64_t row = t * 128 + lb + lane;
#pragma unroll
    for (int cc = 0; cc < 64; cc += 32) {
      float v[32];
      tmem_ld32(tmem + (uint32_t)((j & 1) * 128 + col0 + cc) + ((uint32_t)lb << 16), v);
      if (row < a.rows) {
        const int c0 = col0 + cc;
        if (a.epi == EPI_BIAS_ACT) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float z = v[i] + sbias[c0 + i];
            v[i] = z > 0.f ? z : z * a.alpha;
          }
        } else if (a.epi == EPI_ACT_GRAD) {
          const float4* hp = reinterpret_cast<const float4*>(a.Hprev + row * 128 + c0);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 h = __ldg(hp + i);
            v[4 * i + 0] *= h.x > 0.f ? 1.f : a.alpha;
            v[4 * i + 1] *= h.y > 0.f ? 1.f : a.alpha;
            v[4 * i + 2] *= h.z > 0.f ? 1.f : a.alpha;
            v[4 * i + 3] *= h.w > 0.f ? 1.f : a.alpha;
          }
        }
        float4* cp = reinterpret_cast<float4*>(a.C + row * 128 + c0);
#pragma unroll
        for (int i = 0; i < 8; ++i) cp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    }
    tc_fence_before();
  };

  for (int i = 0; i < nmine; ++i) {
    const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
    uint8_t* sa = sA + (i & 1) * P * kTile;
    stage_rows<kSplit, 128>(a.A, 128, t * 128, a.rows, sa, sa + kTile);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)((i & 1) * 128);
      const uint32_t ah = smem_u32(sa), al = smem_u32(sa + kTile);
      const uint32_t bh = smem_u32(sW), bl = smem_u32(sW + kTile);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t aoff = (k >> 2) * 16384 + (k & 3) * 32;
        uint32_t boff, blbo;
        if (kDgrad) { boff = k * 2048; blbo = 16384; } else { boff = aoff; blbo = 16; }
        const uint64_t adh = make_desc(ah + aoff, 16, 1024);
        const uint64_t bdh = make_desc(bh + boff, blbo, 1024);
        mma_bf16(d, adh, bdh, idesc, k > 0);
        if (kSplit) {
          mma_bf16(d, adh, make_desc(bl + boff, blbo, 1024), idesc, 1);
          mma_bf16(d, make_desc(al + aoff, 16, 1024), bdh, idesc, 1);
        }
      }
      mma_commit(&bar[i & 1]);
    }
    if (i > 0) epilogue(i - 1);
  }
  if (nmine > 0) epilogue(nmine - 1);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// ---------------------------------------------------------------- wgrad
struct WgradArgs {
  const float* dZ;   // [rows][128 out]
  const float* H;    // [rows][128 in]
  int64_t rows;
  int64_t rows_per_cta;
  float* part;       // [grid][128][128]
  float* part_db;    // [grid][128]
};

template <bool kSplit>
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_wgrad(WgradArgs a) {
  constexpr int RB = kSplit ? 64 : 128;          // rows per K block
  constexpr uint32_t kBlk = RB * 128 * 2;        // one [RB][128] bf16 tile
  constexpr int P = kSplit ? 2 : 1;
  constexpr uint32_t kStage = 2 * P * kBlk;      // dZ planes + H planes
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStage = base;                        // 2 stages
  uint8_t* sOnes = base + 2 * kStage;            // [16][RB] ones, SW128 K-major
  constexpr uint32_t kOnes = 16 * RB * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sOnes + kOnes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  for (int i = tid; i < (int)(kOnes / 16); i += blockDim.x) {
    const uint32_t one2 = pack_bf16(1.f, 1.f);
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(one2, one2, one2, one2);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t acc_w = tmem, acc_b = tmem + 128;

  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r1 = min(a.rows, r0 + a.rows_per_cta);
  const int nblk = r1 > r0 ? (int)((r1 - r0 + RB - 1) / RB) : 0;
  constexpr uint32_t idw = make_idesc_bf16(128, 128, 1, 1);
  constexpr uint32_t idb = make_idesc_bf16(128, 16, 1, 0);
  constexpr uint32_t kRegion = RB * 128;         // bytes per 64-column region

  for (int b = 0; b < nblk; ++b) {
    uint8_t* st = sStage + (b & 1) * kStage;
    if (b >= 2) mbar_wait(&bar[b & 1], ((b - 2) >> 1) & 1);
    const int64_t rb = r0 + (int64_t)b * RB;
    stage_rows<kSplit, RB>(a.dZ, 128, rb, r1, st, st + kBlk);
    stage_rows<kSplit, RB>(a.H, 128, rb, r1, st + P * kBlk, st + P * kBlk + kBlk);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t zh = smem_u32(st), zl = smem_u32(st + kBlk);
      const uint32_t hh = smem_u32(st + P * kBlk), hl = smem_u32(st + P * kBlk + kBlk);
      const uint32_t on = smem_u32(sOnes);
#pragma unroll
      for (int k = 0; k < RB / 16; ++k) {
        const uint32_t koff = k * 2048;            // 16 rows = 2 groups of 8
        const uint32_t ooff = (k >> 2) * (16 * 128) + (k & 3) * 32;
        const uint32_t acc0 = (b > 0 || k > 0) ? 1u : 0u;
        const uint64_t zdh = make_desc(zh + koff, kRegion, 1024);
        const uint64_t hdh = make_desc(hh + koff, kRegion, 1024);
        const uint64_t od = make_desc(on + ooff, 16, 1024);
        mma_bf16(acc_w, zdh, hdh, idw, acc0);
        mma_bf16(acc_b, zdh, od, idb, acc0);
        if (kSplit) {
          const uint64_t zdl = make_desc(zl + koff, kRegion, 1024);
          mma_bf16(acc_w, zdh, make_desc(hl + koff, kRegion, 1024), idw, 1);
          mma_bf16(acc_w, zdl, hdh, idw, 1);
          mma_bf16(acc_b, zdl, od, idb, 1);
        }
      }
      mma_commit(&bar[b & 1]);
    }
  }
  // drain: the last commit covers every MMA issued before it
  const int o = 32 * (warp & 3) + lane;           // TMEM lane = output feature
  const int col0 = 64 * (warp >> 2);
  float* dst = a.part + (int64_t)blockIdx.x * 128 * 128 + (int64_t)o * 128 + col0;
  if (nblk > 0) {
    mbar_wait(&bar[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int cc = 0; cc < 64; cc += 32) {
      float v[32];
      tmem_ld32(acc_w + (uint32_t)(col0 + cc) + ((uint32_t)(32 * (warp & 3)) << 16), v);
      float4* p = reinterpret_cast<float4*>(dst + cc);
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
    if (warp < 4) {
      float v[32];
      tmem_ld32(acc_b + ((uint32_t)(32 * warp) << 16), v);
      a.part_db[(int64_t)blockIdx.x * 128 + o] = v[0];
    }
  } else {
    float4* p = reinterpret_cast<float4*>(dst);
    for (int i = 0; i < 16; ++i) p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (warp < 4) a.part_db[(int64_t)blockIdx.x * 128 + o] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// ---------------------------------------------------------------- host
static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
    g_num_sms = std::min(g_num_sms, kMaxSms);
  }
  return g_num_sms;
}

static size_t rows_smem(bool split) {
  const int P = split ? 2 : 1;
  return 1024 + (size_t)3 * P * kTile + 64 + 512;
}
static size_t wgrad_smem(bool split) {
  const int RB = split ? 64 : 128;
  const int P = split ? 2 : 1;
  return 1024 + (size_t)2 * 2 * P * RB * 128 * 2 + 16 * RB * 2 + 64;
}

template <typename K>
static void set_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void tc_configure() {
  static bool done = false;
  if (done) return;
  done = true;
  set_smem(k_tc_rows<true, false>, rows_smem(true));
  set_smem(k_tc_rows<true, true>, rows_smem(true));
  set_smem(k_tc_rows<false, false>, rows_smem(false));
  set_smem(k_tc_rows<false, true>, rows_smem(false));
  set_smem(k_tc_wgrad<true>, wgrad_smem(true));
  set_smem(k_tc_wgrad<false>, wgrad_smem(false));
}

void launch_tc_rows(bool split, bool dgrad, const float* A, const float* W, float* C, int64_t rows, int epi,
                    const float* bias, const float* Hprev, float alpha, cudaStream_t st) {
  if (rows <= 0) return;
  tc_configure();
  RowsArgs a{A, W, C, rows, bias, Hprev, alpha, epi};
  const int64_t ntiles = (rows + 127) / 128;
  const int grid = (int)std::min<int64_t>(ntiles, num_sms());
  const size_t sm = rows_smem(split);
  if (split) {
    if (dgrad) k_tc_rows<true, true><<<grid, kTcThreads, sm, st>>>(a);
    else k_tc_rows<true, false><<<grid, kTcThreads, sm, st>>>(a);
  } else {
    if (dgrad) k_tc_rows<false, true><<<grid, kTcThreads, sm, st>>>(a);
    else k_tc_rows<false, false><<<grid, kTcThreads, sm, st>>>(a);
  }
  count_launch();
}

int tc_wgrad_grid() { return num_sms(); }

void launch_tc_wgrad(bool split, const float* dZ, const float* H, int64_t rows, float* part, float* part_db,
                     cudaStream_t st) {
  tc_configure();
  const int grid = tc_wgrad_grid();
  const int RB = split ? 64 : 128;
  int64_t rpc = (rows + grid - 1) / grid;
  rpc = ((rpc + RB - 1) / RB) * RB;
  WgradArgs a{dZ, H, rows, rpc, part, part_db};
  if (split) k_tc_wgrad<true><<<grid, kTcThreads, wgrad_smem(true), st>>>(a);
  else k_tc_wgrad<false><<<grid, kTcThreads, wgrad_smem(false), st>>>(a);
  count_launch();
}

}  // namespace sagips
