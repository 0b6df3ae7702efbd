// k_data.cu -- random-number-driven kernels of the step: Kaiming init,
// reference data, bootstrap shard, generator noise, the fused event sampler
// (constrain -> Philox -> inverse CDF -> feature rows -> histograms, plus the
// bootstrap gather of the real rows), and the sampler backward.
//
// Paper: P:272 (reference data from known parameters), P:144-146 + P:387
// (50% shard, bootstrap batches), P:295 (inverse-CDF sampler), P:297 (Kaiming
// normal init).  Readings R1, R-RNG, R-UNIF, R-BOOT, R22 in DESIGN.md.
#include "internal.h"

namespace sagips {

// ---------------------------------------------------------------- normals
// Call c of the stream gives normals 4c..4c+3: (w0,w1) -> (r cos, r sin),
// (w2,w3) -> (r cos, r sin), r = sqrt(-2 ln u_a), angle 2 pi u_b.
__global__ void k_normals(float* __restrict__ out, int64_t count, float scale, PhiloxKey key,
                          uint32_t step, uint32_t rank, uint32_t stream) {
  const int64_t ncalls = (count + 3) / 4;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncalls;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox_call(key, (uint32_t)c, step, rank, stream);
    float z[4];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const float ua = uniform_open01(p ? w.z : w.x);
      const float ub = uniform_open01(p ? w.w : w.y);
      const float r = sqrtf(-2.0f * logf(ua));
      float s, co;
      sincospif(2.0f * ub, &s, &co);
      z[2 * p] = r * co;
      z[2 * p + 1] = r * s;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t f = 4 * c + q;
      if (f < count) out[f] = scale * z[q];
    }
  }
}

void launch_normals(float* out, int64_t count, float scale, uint64_t seed, uint32_t step,
                    uint32_t rank, uint32_t stream_id, cudaStream_t st) {
  if (count <= 0) return;
  const int64_t ncalls = (count + 3) / 4;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((ncalls + threads - 1) / threads, 148 * 16);
  k_normals<<<blocks, threads, 0, st>>>(out, count, scale, make_key(seed), step, rank, stream_id);
  count_launch();
}

// ---------------------------------------------------------------- reference
// ref[i][o] = Q(u(word 2i+o of stream REF, step 0, rank 0); c_true[o]).
__global__ void k_reference(float* __restrict__ ref, int64_t n, Coef6 c, PhiloxKey key) {
  const int64_t ncalls = (n + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ncalls;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox_call(key, (uint32_t)q, 0, 0, kStreamRef);
    const int64_t e0 = 2 * q;
    ref[2 * e0 + 0] = quantile_f32(uniform_open01(w.x), c.v[0], c.v[1], c.v[2]);
    ref[2 * e0 + 1] = quantile_f32(uniform_open01(w.y), c.v[3], c.v[4], c.v[5]);
    if (e0 + 1 < n) {
      ref[2 * e0 + 2] = quantile_f32(uniform_open01(w.z), c.v[0], c.v[1], c.v[2]);
      ref[2 * e0 + 3] = quantile_f32(uniform_open01(w.w), c.v[3], c.v[4], c.v[5]);
    }
  }
}

void launch_reference(float* ref, int64_t n, const float c_true[6], uint64_t seed, cudaStream_t st) {
  Coef6 c;
  for (int i = 0; i < 6; ++i) c.v[i] = c_true[i];
  const int64_t ncalls = (n + 1) / 2;
  const int blocks = (int)std::min<int64_t>((ncalls + 255) / 256, 148 * 16);
  k_reference<<<blocks, 256, 0, st>>>(ref, n, c, make_key(seed));
  count_launch();
}

// ---------------------------------------------------------------- shard
// shard[i] = ref[(w_i * n_ref) >> 32], w_i = word i of stream SHARD (step 0).
__global__ void k_shard(const float2* __restrict__ ref, uint32_t n_ref, float2* __restrict__ shard,
                        int64_t n_s, PhiloxKey key, uint32_t rank) {
  const int64_t ncalls = (n_s + 3) / 4;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncalls;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox_call(key, (uint32_t)c, 0, rank, kStreamShard);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = 4 * c + q;
      if (i < n_s) shard[i] = ref[lemire(word_of(w, q), n_ref)];
    }
  }
}

void launch_shard(const float* ref, int64_t n_ref, float* shard, int64_t n_s, uint64_t seed,
                  uint32_t rank, cudaStream_t st) {
  const int64_t ncalls = (n_s + 3) / 4;
  const int blocks = (int)std::min<int64_t>((ncalls + 255) / 256, 148 * 16);
  k_shard<<<blocks, 256, 0, st>>>(reinterpret_cast<const float2*>(ref), (uint32_t)n_ref,
                                  reinterpret_cast<float2*>(shard), n_s, make_key(seed), rank);
  count_launch();
}

// ---------------------------------------------------------------- constrain
// c[s] = (raw0, softplus(raw1), softplus(raw2), raw3, softplus(raw4), softplus(raw5)) (R1);
// tabulated sampler (R32): (sigmoid(raw0), softplus(raw1), softplus(raw2), ...) = (w, b, c) per observable
__global__ void k_constrain(const float* __restrict__ raw, float* __restrict__ c, int k, int tab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 6 * k) return;
  const int j = i % 3;
  const float x = raw[i];
  c[i] = (j == 0) ? (tab ? sigmoid_f(x) : x) : softplus_f(x);
}

void launch_constrain(const float* raw, float* c, int k, cudaStream_t st, bool tab) {
  k_constrain<<<(6 * k + 255) / 256, 256, 0, st>>>(raw, c, k, tab ? 1 : 0);
  count_launch();
}

// ---------------------------------------------------------------- sampler
// Packed fp32 pairs (sm_100a FADD2 / FMUL2): each lane rounded exactly as the
// scalar instruction, one issue slot per pair -- the two observables of an
// event travel together.
__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk(uint64_t r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fadd2_rm(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// the bits of 1 + (w >> 9) 2^-23 (uniform_open01) as one IMAD.HI on the FMA
// pipe: hi(w * 2^23) + 0x3F800000 = (w >> 9) | 0x3F800000 (w >> 9 < 2^23)
__device__ __forceinline__ uint32_t one_plus_bits(uint32_t w) {
  uint32_t r;
  asm("mad.hi.u32 %0, %1, 8388608, 1065353216;" : "=r"(r) : "r"(w));
  return r;
}
// (u(wa), u(wb)) of R-UNIF, bitwise equal to uniform_open01 on each word
__device__ __forceinline__ uint64_t uniform2(uint32_t wa, uint32_t wb) {
  const uint64_t one_m = pk(__uint_as_float(one_plus_bits(wa)), __uint_as_float(one_plus_bits(wb)));
  return fsub2(one_m, pk(0.99999994039535522461f, 0.99999994039535522461f));
}
// ptxas (CUDA 12.9) contracts mul.rn.f32x2 followed by add.rn.f32x2 into
// FFMA2 -- even with -fmad=false and explicit .rn, unlike the scalar
// instructions -- which would round u c2 + c1 once instead of twice.  An
// XOR of the product's low word with a runtime zero (a kernel argument)
// hides the producer from that peephole: one ALU op, bits unchanged.
__device__ __forceinline__ uint64_t opaque(uint64_t x, uint32_t zero) {
  uint64_t r;
  asm("{.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\txor.b32 lo, lo, %2;\n\tmov.b64 %0, {lo, hi};}"
      : "=l"(r) : "l"(x), "r"(zero));
  return r;
}
// Q(u; c) of both observables (quantile_f32 per lane: four separately
// rounded operations): c0 + u (c1 + u c2) with C_j = (c_j of observable 0,
// c_j of observable 1)
__device__ __forceinline__ uint64_t quantile2(uint64_t u, uint64_t C0, uint64_t C1, uint64_t C2, uint32_t zero) {
  const uint64_t b = fadd2(C1, opaque(fmul2(u, C2), zero));
  return fadd2(C0, opaque(fmul2(u, b), zero));
}

// Histogram bins of both observables (hist_bin per lane): t = (y - lo) sc,
// clamp to [-1, bins], floor via the 1.5 * 2^23 rounding trick, + 1.
__device__ __forceinline__ void bins2(uint64_t y, uint64_t LO, uint64_t SC, float fb, int& b0, int& b1) {
  const float2 t = upk(fmul2(fsub2(y, LO), SC));
  const float c0 = fminf(fmaxf(t.x, -1.0f), fb), c1 = fminf(fmaxf(t.y, -1.0f), fb);
  const float2 r = upk(fadd2_rm(pk(c0, c1), pk(12582912.0f, 12582912.0f)));
  b0 = __float_as_int(r.x) - 0x4B400000 + 1;
  b1 = __float_as_int(r.y) - 0x4B400000 + 1;
}

// Shared histograms of a block: [4 = (real, fake) x obs][bins+2][32 lanes]
// uint32 (lane-column layout: lane l of every warp increments column l, so
// one ATOMS of a warp touches 32 distinct banks -- no intra-warp conflicts
// however concentrated the distribution; warps meet only across
// instructions).  Used when 512 (bins+2) bytes fit (bins <= 126); otherwise
// one [4][bins+2] copy per block.
#ifndef SAGIPS_SAMPLE_THREADS
#define SAGIPS_SAMPLE_THREADS 512
#endif
constexpr int kSampleThreads = SAGIPS_SAMPLE_THREADS;
// resident blocks per SM (3 blocks at 40 registers for the variants that do
// not spill then measured no faster at 2^24: 34.4 vs 32.8 us)
#ifndef SAGIPS_SAMPLE_BPS
#define SAGIPS_SAMPLE_BPS 1  // one 512-thread block per SM (2 blocks: 45.5 vs 43.5 us at 2^24 with histograms)
#endif
__host__ __device__ constexpr int sample_blocks_per_sm(bool, bool, bool) { return SAGIPS_SAMPLE_BPS; }
__host__ __device__ constexpr bool hist_columns(int bins) { return bins + 2 <= 128; }

// One thread = one group of 4 consecutive events e = 4g..4g+3:
//   fake: Philox calls 2g and 2g+1 of stream FAKE give the 8 words 2e+o;
//   real: call g of stream REAL gives the 4 bootstrap words (word e).
// Rows of X: [0, N) real, [N, 2N) fake (R9).  Persistent grid (2 blocks of
// 512 per SM), grid-stride over groups; the common group (all 4 events in
// range and in one sample, 16-B aligned rows) runs a branch-free body with
// FADD2/FMUL2 pairs; the ragged tail and m % 4 != 0 take the general one.
// Histograms: see hist_columns; per block one merge into the global counts
// with integer atomics (exact, order-independent).
// kFake = false: the real rows only (the tabulated sampler, R32, draws the fake rows)
template <bool kReal, bool kHist, bool kFake = true>
__global__ void __launch_bounds__(kSampleThreads, sample_blocks_per_sm(kReal, kHist, kFake))
    k_sample(const float* __restrict__ c, int m, int64_t n_events, const float2* __restrict__ shard,
             uint32_t n_shard, PhiloxKey key, uint32_t step, uint32_t rank, uint32_t fake_stream,
             float2* __restrict__ x_real, float2* __restrict__ y_fake, uint32_t* __restrict__ real_idx,
             uint32_t* __restrict__ hist, int bins, float lo0, float sc0, float lo1, float sc1, int vec_ok,
             uint32_t zero) {
  extern __shared__ uint32_t sh_hist[];
  const int nb = bins + 2;
  const bool cols = hist_columns(bins);
  const int hwords = 4 * nb * (cols ? 32 : 1);
  const int lane = threadIdx.x & 31;
  if (kHist) {
    for (int i = threadIdx.x; i < hwords; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
  }
  // word offset of counter (h, bin) for this thread: (h nb + bin) 32 + lane, or h nb + bin
  const int hstride = cols ? 32 : 1;
  uint32_t* hbase = sh_hist + (cols ? lane : 0);
  auto hadd = [&](int h, int bin) { atomicAdd(hbase + (h * nb + bin) * hstride, 1u); };
  const float fb = (float)bins;
  const uint64_t LO = pk(lo0, lo1), SC = pk(sc0, sc1);
  // event counts are < 2^31 (validated at the ABI), so 32-bit indices
  const uint32_t n = (uint32_t)n_events;
  const uint32_t ngroups = (n + 3) / 4;
  const bool m4 = (m & 3) == 0 && vec_ok;
  const PhiloxRoundKeys rk = round_keys(key);
  // sample of the group's first event, s = 4g / m, and its offset r in the
  // sample: two divisions per thread, then advanced by the grid stride
  const uint32_t g0 = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  const uint32_t um = (uint32_t)m, ds = 4 * gstride / um, dr = 4 * gstride - ds * um;
  uint32_t s = 4 * g0 / um, r0 = 4 * g0 - s * um;
  for (uint32_t g = g0; g < ngroups; g += gstride, s += ds, r0 += dr, (r0 >= um ? (r0 -= um, ++s) : 0u)) {
    uint4 wa = make_uint4(0, 0, 0, 0), wb = make_uint4(0, 0, 0, 0);
    if (kFake) {
      wa = philox4x32_10(make_uint4(2 * g, step, rank, fake_stream), rk);
      wb = philox4x32_10(make_uint4(2 * g + 1, step, rank, fake_stream), rk);
    }
    const uint32_t wf[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
    uint4 wr = make_uint4(0, 0, 0, 0);
    if (kReal) wr = philox4x32_10(make_uint4(g, step, rank, kStreamReal), rk);
    const float* cs = c + 6 * (size_t)s;
    uint64_t C0 = 0, C1 = 0, C2 = 0;
    auto load_c = [&]() {
      C0 = pk(__ldg(cs + 0), __ldg(cs + 3));
      C1 = pk(__ldg(cs + 1), __ldg(cs + 4));
      C2 = pk(__ldg(cs + 2), __ldg(cs + 5));
    };
    if (kFake) load_c();
    float2 yv[4], xv[4];
    uint32_t iv[4];
    if (kReal) {
#pragma unroll
      for (int q = 0; q < 4; ++q) iv[q] = lemire(word_of(wr, q), n_shard);
    }
    auto event = [&](int q) {
      if (kFake) {
        const uint64_t y = quantile2(uniform2(wf[2 * q], wf[2 * q + 1]), C0, C1, C2, zero);
        yv[q] = upk(y);
        if (kHist) {
          int b0, b1;
          bins2(y, LO, SC, fb, b0, b1);
          hadd(2, b0);
          hadd(3, b1);
        }
      }
      if (kReal) {
        xv[q] = __ldg(shard + iv[q]);
        if (kHist) {
          int b0, b1;
          bins2(pk(xv[q].x, xv[q].y), LO, SC, fb, b0, b1);
          hadd(0, b0);
          hadd(1, b1);
        }
      }
    };
    if (m4 && 4 * g + 3 < n) {
#pragma unroll
      for (int q = 0; q < 4; ++q) event(q);
      if (kFake) {
        float4* yf = reinterpret_cast<float4*>(y_fake + 4 * (size_t)g);
        __stcs(yf, make_float4(yv[0].x, yv[0].y, yv[1].x, yv[1].y));
        __stcs(yf + 1, make_float4(yv[2].x, yv[2].y, yv[3].x, yv[3].y));
      }
      if (kReal) {
        float4* xr = reinterpret_cast<float4*>(x_real + 4 * (size_t)g);
        __stcs(xr, make_float4(xv[0].x, xv[0].y, xv[1].x, xv[1].y));
        __stcs(xr + 1, make_float4(xv[2].x, xv[2].y, xv[3].x, xv[3].y));
        __stcs(reinterpret_cast<uint4*>(real_idx + 4 * (size_t)g), make_uint4(iv[0], iv[1], iv[2], iv[3]));
      }
    } else {
      // general group: step across sample boundaries, stop at n
      uint32_t r = r0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t e = 4 * g + q;
        if (e >= n) break;
        if (r == (uint32_t)m) {
          r = 0;
          cs += 6;
          if (kFake) load_c();
        }
        ++r;
        event(q);
        if (kFake) y_fake[e] = yv[q];
        if (kReal) {
          x_real[e] = xv[q];
          real_idx[e] = iv[q];
        }
      }
    }
  }
  if (kHist) {
    __syncthreads();
    const int h0 = kReal ? 0 : 2, h1 = kFake ? 4 : 2;  // histograms this launch fills
    for (int i = h0 * nb + threadIdx.x; i < h1 * nb; i += blockDim.x) {
      uint32_t v = 0;
      if (cols) {
        const uint4* p = reinterpret_cast<const uint4*>(sh_hist + i * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 q = p[(j + threadIdx.x) & 7];  // rotated start: spread the banks
          v += q.x + q.y + q.z + q.w;
        }
      } else {
        v = sh_hist[i];
      }
      if (v) atomicAdd(&hist[i - (kReal ? 0 : 2 * nb)], v);
    }
  }
}

static void hist_params(const float lo[2], const float hi[2], int bins, float* sc) {
  for (int o = 0; o < 2; ++o) sc[o] = (float)bins / (hi[o] - lo[o]);  // fp32, as the oracle
}

// persistent launch shape: up to 2 blocks of 512 per SM (all SMs busy: at
// 2^20 events, ~1.7 groups per thread; the kernel is latency-bound there --
// ncu: 25% occupancy and 35% idle SM cycles with 128 blocks)
static int g_sm_count = 0;
static int sm_count() {
  if (!g_sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  return g_sm_count;
}
static void sample_shape(int64_t n, int bins, bool hist, int bps, int* blocks, size_t* smem) {
  const int64_t ngroups = (n + 3) / 4;
  const int64_t want = (ngroups + kSampleThreads - 1) / kSampleThreads;
  *blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, bps * (int64_t)sm_count()));
  *smem = hist ? sizeof(uint32_t) * 4 * (bins + 2) * (hist_columns(bins) ? 32 : 1) : 0;
}

template <bool R, bool H, bool F>
static void set_smem_attr(size_t smem) {
  static size_t done = 0;
  if (smem > 48 * 1024 && smem > done) {
    cudaFuncSetAttribute(k_sample<R, H, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    done = smem;
  }
}

void launch_sample_step(const float* c, int k, int m, const float* shard, int64_t n_shard,
                        uint64_t seed, uint32_t step, uint32_t rank, float* x_events,
                        uint32_t* real_idx, uint32_t* hist, int bins, const float lo[2],
                        const float hi[2], cudaStream_t st, bool fake, bool hist_zeroed) {
  const int64_t n = (int64_t)k * m;
  float sc[2];
  hist_params(lo, hi, bins, sc);
  if (hist && !hist_zeroed) cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 4 * (bins + 2), st);
  int blocks;
  size_t smem;
  sample_shape(n, bins, hist != nullptr, sample_blocks_per_sm(true, hist != nullptr, fake), &blocks, &smem);
  float2* x = reinterpret_cast<float2*>(x_events);
  const int vec_ok = (n % 2 == 0) && (reinterpret_cast<uintptr_t>(x_events) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(real_idx) % 16 == 0);
  auto kern = fake ? (hist ? k_sample<true, true> : k_sample<true, false>)
                   : (hist ? k_sample<true, true, false> : k_sample<true, false, false>);
  if (fake && hist) set_smem_attr<true, true, true>(smem);
  if (!fake && hist) set_smem_attr<true, true, false>(smem);
  kern<<<blocks, kSampleThreads, smem, st>>>(c, m, n, reinterpret_cast<const float2*>(shard), (uint32_t)n_shard,
                                             make_key(seed), step, rank, kStreamFake, x, x + n, real_idx, hist, bins,
                                             lo[0], sc[0], lo[1], sc[1], vec_ok, 0u);
  count_launch();
}

void launch_sample_events(const float* c, int k, int m, uint64_t seed, uint32_t step, uint32_t rank,
                          uint32_t stream_id, float* events, uint32_t* hist, int bins,
                          const float lo[2], const float hi[2], cudaStream_t st) {
  const int64_t n = (int64_t)k * m;
  float sc[2] = {0.f, 0.f};
  float l[2] = {0.f, 0.f};
  if (hist) {
    hist_params(lo, hi, bins, sc);
    l[0] = lo[0];
    l[1] = lo[1];
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 2 * (bins + 2), st);
  }
  int blocks;
  size_t smem;
  sample_shape(n, bins, hist != nullptr, sample_blocks_per_sm(false, hist != nullptr, true), &blocks, &smem);
  const int vec_ok = reinterpret_cast<uintptr_t>(events) % 16 == 0;
  auto kern = hist ? k_sample<false, true> : k_sample<false, false>;
  if (hist) set_smem_attr<false, true, true>(smem);
  kern<<<blocks, kSampleThreads, smem, st>>>(c, m, n, nullptr, 1, make_key(seed), step, rank, stream_id, nullptr,
                                             reinterpret_cast<float2*>(events), nullptr, hist, bins, l[0], sc[0], l[1],
                                             sc[1], vec_ok, 0u);
  count_launch();
}

// ---------------------------------------------------------------- sampler backward
// One block per parameter sample s:
//   dc[o][j] = sum_{e in s} dy[e][o] * u[e][o]^j   (dQ/dc = (1, u, u^2))
//   draw[s][3o] = dc[o][0], draw[s][3o+1] = dc[o][1] softplus'(raw), ...
// u is recomputed from the FAKE stream (not stored): one Philox call serves
// the event pair 2q, 2q+1 (words 0,1 and 2,3), so a thread takes pairs when
// the sample starts on an even event (m even), else single events.  The
// block reduction has a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) k_sample_bwd(const float2* __restrict__ dy, const float* __restrict__ raw,
                                                    int m, PhiloxKey key, uint32_t step, uint32_t rank,
                                                    float* __restrict__ draw, const __grid_constant__ LossFinish loss) {
  if (loss.loss_part && blockIdx.x == gridDim.x - 1) {  // the extra block: the step's G loss
    __shared__ double sp[kLossCap];
    finish_loss_block(loss.loss_part, loss.nparts, loss.scale, loss.out, loss.nonfinite, sp);
    return;
  }
  const int s = blockIdx.x;
  float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto add = [&](float2 g, float u0, float u1) {
    acc[0] += g.x;
    acc[1] += g.x * u0;
    acc[2] += g.x * u0 * u0;
    acc[3] += g.y;
    acc[4] += g.y * u1;
    acc[5] += g.y * u1 * u1;
  };
  const int64_t e0 = (int64_t)s * m;
  if ((m & 1) == 0) {
    const PhiloxRoundKeys rk = round_keys(key);
    for (int i = 2 * threadIdx.x; i < m; i += 2 * blockDim.x) {
      const int64_t e = e0 + i;
      const uint4 w = philox4x32_10(make_uint4((uint32_t)(e >> 1), step, rank, kStreamFake), rk);
      const float4 g = __ldcs(reinterpret_cast<const float4*>(dy + e));
      add(make_float2(g.x, g.y), uniform_open01(w.x), uniform_open01(w.y));
      add(make_float2(g.z, g.w), uniform_open01(w.z), uniform_open01(w.w));
    }
  } else {
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const int64_t e = e0 + i;
      const uint4 w = philox_call(key, (uint32_t)(e >> 1), step, rank, kStreamFake);
      const bool odd = e & 1;
      add(dy[e], uniform_open01(odd ? w.z : w.x), uniform_open01(odd ? w.w : w.y));
    }
  }
  __shared__ float red[6][32];
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    float v = acc[j];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) red[j][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int j = threadIdx.x;
    float v = 0.f;
    for (int wi = 0; wi < (int)(blockDim.x >> 5); ++wi) v += red[j][wi];
    const int jj = j % 3;
    const float r = raw[6 * s + j];
    draw[6 * s + j] = jj == 0 ? v : v * softplus_grad_f(r);
  }
}

void launch_sample_bwd(const float* dy, const float* raw, int k, int m, uint64_t seed, uint32_t step,
                       uint32_t rank, float* draw, cudaStream_t st, const LossFinish& loss) {
  const int per = (m % 2 == 0) ? (m + 1) / 2 : m;  // work items per sample
  int threads = 32 * ((std::min(per, 256) + 31) / 32);
  k_sample_bwd<<<k + (loss.loss_part ? 1 : 0), threads, 0, st>>>(reinterpret_cast<const float2*>(dy), raw, m,
                                                                  make_key(seed), step, rank, draw, loss);
  count_launch();
}

}  // namespace sagips
