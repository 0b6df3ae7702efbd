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
// One thread = one group of 4 consecutive events e = 4g..4g+3:
//   fake: Philox calls 2g and 2g+1 of stream FAKE give the 8 words 2e+o;
//   real: call g of stream REAL gives the 4 bootstrap words (word e).
// Histogram increment (shared-memory atomic into the warp's private copy).
__device__ __forceinline__ void hist_add(uint32_t* h, int bin) { atomicAdd(h + bin, 1u); }

// Rows of X: [0, N) real, [N, 2N) fake (R9).  Persistent grid (grid-stride
// over groups).  Histograms are privatised per warp in shared memory when they
// fit (no inter-warp contention), summed per block, and merged with integer
// atomics (exact and order-independent).  The common group (all 4 events in
// range and in one sample, 16-B aligned rows) runs a branch-free body; the
// ragged tail and m % 4 != 0 take the general one.
// kFake = false: the real rows only (the tabulated sampler, R32, draws the fake rows)
template <bool kReal, bool kHist, bool kFake = true>
__global__ void __launch_bounds__(256) k_sample(const float* __restrict__ c, int m, int64_t n_events,
                                                const float2* __restrict__ shard, uint32_t n_shard,
                                                PhiloxKey key, uint32_t step, uint32_t rank,
                                                uint32_t fake_stream, float2* __restrict__ x_real,
                                                float2* __restrict__ y_fake, uint32_t* __restrict__ real_idx,
                                                uint32_t* __restrict__ hist, int bins, float lo0, float sc0,
                                                float lo1, float sc1, int per_warp, int vec_ok) {
  extern __shared__ uint32_t sh_hist[];  // [copies][2 sets][2 obs][bins+2]
  const int hsz = 4 * (bins + 2);
  const int copies = per_warp ? (int)(blockDim.x >> 5) : 1;
  uint32_t* my = sh_hist + (per_warp ? (int)(threadIdx.x >> 5) * hsz : 0);
  if (kHist) {
    for (int i = threadIdx.x; i < hsz * copies; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
  }
  // event counts are < 2^31 (validated at the ABI), so 32-bit indices
  const uint32_t n = (uint32_t)n_events;
  const uint32_t ngroups = (n + 3) / 4;
  const bool m4 = (m & 3) == 0 && vec_ok;
  uint32_t* hx0 = my;
  uint32_t* hx1 = my + (bins + 2);
  uint32_t* hy0 = my + 2 * (bins + 2);
  uint32_t* hy1 = my + 3 * (bins + 2);
  const PhiloxRoundKeys rk = round_keys(key);
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
    uint4 wa = make_uint4(0, 0, 0, 0), wb = make_uint4(0, 0, 0, 0);
    if (kFake) {
      wa = philox4x32_10(make_uint4(2 * g, step, rank, fake_stream), rk);
      wb = philox4x32_10(make_uint4(2 * g + 1, step, rank, fake_stream), rk);
    }
    const uint32_t wf[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
    uint4 wr = make_uint4(0, 0, 0, 0);
    if (kReal) wr = philox4x32_10(make_uint4(g, step, rank, kStreamReal), rk);
    // sample of the group's first event: one division per group
    const uint32_t s = 4 * g / (uint32_t)m;
    const float* cs = c + 6 * (size_t)s;
    float c0 = __ldg(cs + 0), c1 = __ldg(cs + 1), c2 = __ldg(cs + 2);
    float c3 = __ldg(cs + 3), c4 = __ldg(cs + 4), c5 = __ldg(cs + 5);
    float2 yv[4], xv[4];
    uint32_t iv[4];
    auto event = [&](int q) {
      if (kFake) {
        yv[q].x = quantile_f32(uniform_open01(wf[2 * q]), c0, c1, c2);
        yv[q].y = quantile_f32(uniform_open01(wf[2 * q + 1]), c3, c4, c5);
      }
      if (kHist && kFake) {
        hist_add(hy0, hist_bin(yv[q].x, lo0, sc0, bins));
        hist_add(hy1, hist_bin(yv[q].y, lo1, sc1, bins));
      }
      if (kReal) {
        iv[q] = lemire(word_of(wr, q), n_shard);
        xv[q] = __ldg(shard + iv[q]);
        if (kHist) {
          hist_add(hx0, hist_bin(xv[q].x, lo0, sc0, bins));
          hist_add(hx1, hist_bin(xv[q].y, lo1, sc1, bins));
        }
      }
    };
    if (m4 && 4 * g + 3 < n) {
#pragma unroll
      for (int q = 0; q < 4; ++q) event(q);
      if (kFake) {
        float4* yf = reinterpret_cast<float4*>(y_fake + 4 * (size_t)g);
        yf[0] = make_float4(yv[0].x, yv[0].y, yv[1].x, yv[1].y);
        yf[1] = make_float4(yv[2].x, yv[2].y, yv[3].x, yv[3].y);
      }
      if (kReal) {
        float4* xr = reinterpret_cast<float4*>(x_real + 4 * (size_t)g);
        xr[0] = make_float4(xv[0].x, xv[0].y, xv[1].x, xv[1].y);
        xr[1] = make_float4(xv[2].x, xv[2].y, xv[3].x, xv[3].y);
        *reinterpret_cast<uint4*>(real_idx + 4 * (size_t)g) = make_uint4(iv[0], iv[1], iv[2], iv[3]);
      }
    } else {
      // general group: step across sample boundaries, stop at n
      uint32_t r = 4 * g - s * (uint32_t)m;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t e = 4 * g + q;
        if (e >= n) break;
        if (r == (uint32_t)m) {
          r = 0;
          cs += 6;
          c0 = __ldg(cs + 0); c1 = __ldg(cs + 1); c2 = __ldg(cs + 2);
          c3 = __ldg(cs + 3); c4 = __ldg(cs + 4); c5 = __ldg(cs + 5);
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
    const int off = kReal ? 0 : 2 * (bins + 2);
    for (int i = off + threadIdx.x; i < hsz; i += blockDim.x) {
      uint32_t v = 0;
      for (int w = 0; w < copies; ++w) v += sh_hist[w * hsz + i];
      if (v) atomicAdd(&hist[i - off], v);
    }
  }
}

static void hist_params(const float lo[2], const float hi[2], int bins, float* sc) {
  for (int o = 0; o < 2; ++o) sc[o] = (float)bins / (hi[o] - lo[o]);  // fp32, as the oracle
}

// persistent launch shape: 2 blocks per SM; per-warp histogram copies when
// 8 x 4 x (bins+2) counters fit comfortably in shared memory
static void sample_shape(int64_t n, int bins, bool hist, int* blocks, size_t* smem, int* per_warp) {
  const int64_t ngroups = (n + 3) / 4;
  *blocks = (int)std::max<int64_t>(1, std::min<int64_t>((ngroups + 255) / 256, 148 * 8));
  *per_warp = hist && (8 * 4 * (bins + 2) * 4 <= 48 * 1024);
  *smem = hist ? sizeof(uint32_t) * 4 * (bins + 2) * (*per_warp ? 8 : 1) : 0;
}

void launch_sample_step(const float* c, int k, int m, const float* shard, int64_t n_shard,
                        uint64_t seed, uint32_t step, uint32_t rank, float* x_events,
                        uint32_t* real_idx, uint32_t* hist, int bins, const float lo[2],
                        const float hi[2], cudaStream_t st, bool fake) {
  const int64_t n = (int64_t)k * m;
  float sc[2];
  hist_params(lo, hi, bins, sc);
  if (hist) cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 4 * (bins + 2), st);
  int blocks, per_warp;
  size_t smem;
  sample_shape(n, bins, hist != nullptr, &blocks, &smem, &per_warp);
  float2* x = reinterpret_cast<float2*>(x_events);
  const int vec_ok = (n % 2 == 0) && (reinterpret_cast<uintptr_t>(x_events) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(real_idx) % 16 == 0);
  auto kern = fake ? (hist ? k_sample<true, true> : k_sample<true, false>)
                   : (hist ? k_sample<true, true, false> : k_sample<true, false, false>);
  kern<<<blocks, 256, smem, st>>>(c, m, n, reinterpret_cast<const float2*>(shard),
                                            (uint32_t)n_shard, make_key(seed), step, rank, kStreamFake,
                                            x, x + n, real_idx, hist, bins, lo[0], sc[0], lo[1], sc[1], per_warp,
                                            vec_ok);
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
  int blocks, per_warp;
  size_t smem;
  sample_shape(n, bins, hist != nullptr, &blocks, &smem, &per_warp);
  const int vec_ok = reinterpret_cast<uintptr_t>(events) % 16 == 0;
  auto kern = hist ? k_sample<false, true> : k_sample<false, false>;
  kern<<<blocks, 256, smem, st>>>(c, m, n, nullptr, 1, make_key(seed), step, rank, stream_id,
                                             nullptr, reinterpret_cast<float2*>(events), nullptr, hist,
                                             bins, l[0], sc[0], l[1], sc[1], per_warp, vec_ok);
  count_launch();
}

// ---------------------------------------------------------------- sampler backward
// One block per parameter sample s:
//   dc[o][j] = sum_{e in s} dy[e][o] * u[e][o]^j   (dQ/dc = (1, u, u^2))
//   draw[s][3o] = dc[o][0], draw[s][3o+1] = dc[o][1] softplus'(raw), ...
// u is recomputed from the FAKE stream (not stored).  The block reduction has
// a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) k_sample_bwd(const float2* __restrict__ dy, const float* __restrict__ raw,
                                                    int m, PhiloxKey key, uint32_t step, uint32_t rank,
                                                    float* __restrict__ draw) {
  const int s = blockIdx.x;
  float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int64_t e = (int64_t)s * m + i;
    const uint4 w = philox_call(key, (uint32_t)(e >> 1), step, rank, kStreamFake);
    const bool odd = e & 1;
    const float u0 = uniform_open01(odd ? w.z : w.x);
    const float u1 = uniform_open01(odd ? w.w : w.y);
    const float2 g = dy[e];
    acc[0] += g.x;
    acc[1] += g.x * u0;
    acc[2] += g.x * u0 * u0;
    acc[3] += g.y;
    acc[4] += g.y * u1;
    acc[5] += g.y * u1 * u1;
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
                       uint32_t rank, float* draw, cudaStream_t st) {
  int threads = 32 * ((std::min(m, 256) + 31) / 32);
  k_sample_bwd<<<k, threads, 0, st>>>(reinterpret_cast<const float2*>(dy), raw, m, make_key(seed),
                                      step, rank, draw);
  count_launch();
}

}  // namespace sagips
