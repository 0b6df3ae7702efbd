// k_tabulated.cu -- the tabulated-CDF sampler variant (SURVEY §8(f) row 1,
// reading R32): per parameter sample s and observable o a density on [0, 1]
//     f(x) = w x^b (1-x)^c + (1-w) x^c (1-x)^b,
//     (w, b, c) = (sigmoid(r0), softplus(r1), softplus(r2)), (r0, r1, r2) = raw[s][3o..3o+2],
// tabulated on G grid points t_i = i / (G-1) with a trapezoid CDF
// F_i = S_i / S_{G-1}, and events x = t_i + (u - F_i) / (F_{i+1} - F_i) Delta
// for the cell i with F_i <= u < F_{i+1}; u from the FAKE Philox stream
// exactly as the quadratic sampler (word 2e+o, R-RNG, R-UNIF).  The backward
// is the exact derivative of this tabulated inverse (R32).  Paper: the
// inverse-CDF method of a realistic, sampler-dominated pipeline
// (P:23).
//
// One CTA per parameter sample: the tables live in shared memory (fp64), the
// trapezoid sums are a chunked block scan, and the sample's m events are
// inverted by binary search in shared memory.  Shared memory: forward 2 G,
// backward 8 G doubles (G <= 2048).
#include "ctx.h"

namespace sagips {

namespace {
constexpr int kTabThreads = 256;
constexpr int kTabMaxG = 2048;

__device__ __forceinline__ double softplus_d(double x) { return x > 20.0 ? x : log1p(exp(x)); }
__device__ __forceinline__ double sigmoid_d(double x) { return 1.0 / (1.0 + exp(-x)); }

struct Wbc {
  double w, b, c;
};
__device__ __forceinline__ Wbc constrain_wbc(const float* r) {
  return Wbc{sigmoid_d((double)r[0]), softplus_d((double)r[1]), softplus_d((double)r[2])};
}

// f and (optionally) df/d(w, b, c) at node t (0 at the ends: b, c > 0)
template <bool kGrad>
__device__ __forceinline__ void node(double t, const Wbc& p, double* f, double* fw, double* fb, double* fc) {
  if (t <= 0.0 || t >= 1.0) {
    *f = 0.0;
    if (kGrad) *fw = *fb = *fc = 0.0;
    return;
  }
  const double lt = log(t), ls = log1p(-t);
  const double e1 = exp(p.b * lt + p.c * ls);  // t^b (1-t)^c
  const double e2 = exp(p.c * lt + p.b * ls);  // t^c (1-t)^b
  *f = p.w * e1 + (1.0 - p.w) * e2;
  if (kGrad) {
    *fw = e1 - e2;
    *fb = p.w * e1 * lt + (1.0 - p.w) * e2 * ls;
    *fc = p.w * e1 * ls + (1.0 - p.w) * e2 * lt;
  }
}

// In-place inclusive scan of the trapezoid increments of the G node values in
// v: v_i <- sum_{j=1..i} (v_{j-1} + v_j) Delta / 2 (v_0 <- 0).  Thread t owns
// a contiguous chunk; chunk totals are scanned across the block (fp64).
__device__ void trapezoid_scan(double* v, int G, double delta, double* s_tot) {
  const int t = threadIdx.x;
  const int chunk = (G + kTabThreads - 1) / kTabThreads;
  const int i0 = t * chunk, i1 = min(G, i0 + chunk);
  double inc[kTabMaxG / kTabThreads];
  double run = 0.0;
#pragma unroll
  for (int q = 0; q < kTabMaxG / kTabThreads; ++q) {
    const int i = i0 + q;
    if (i < i1) run += (i > 0) ? (v[i - 1] + v[i]) * (delta * 0.5) : 0.0;
    inc[q] = run;
  }
  s_tot[t] = run;
  __syncthreads();  // every thread has read its v before any write below
  // exclusive scan of the chunk totals (Hillis-Steele over shared memory)
  for (int off = 1; off < kTabThreads; off <<= 1) {
    const double add = t >= off ? s_tot[t - off] : 0.0;
    __syncthreads();
    s_tot[t] += add;
    __syncthreads();
  }
  const double base = t > 0 ? s_tot[t - 1] : 0.0;
#pragma unroll
  for (int q = 0; q < kTabMaxG / kTabThreads; ++q) {
    const int i = i0 + q;
    if (i < i1) v[i] = base + inc[q];
  }
  __syncthreads();
}

// largest i with F_i <= u, clipped to [0, G-2]
__device__ __forceinline__ int find_cell(const double* F, int G, double u) {
  int lo = 0, hi = G - 1;  // invariant: F[lo] <= u (F[0] = 0 < u), answer in [lo, hi)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (F[mid] <= u) lo = mid;
    else hi = mid;
  }
  return min(lo, G - 2);
}

__device__ __forceinline__ double event_u(PhiloxKey key, uint32_t step, uint32_t rank, uint32_t stream, int64_t e,
                                          int o) {
  const uint64_t word = 2 * (uint64_t)e + o;
  const uint4 r = philox_call(key, (uint32_t)(word >> 2), step, rank, stream);
  return (double)uniform_open01(word_of(r, (int)(word & 3)));
}
}  // namespace

struct TabHist {
  uint32_t* hist;  // [2 obs][bins+2] or nullptr
  int bins;
  float lo0, sc0, lo1, sc1;
};

__global__ void __launch_bounds__(kTabThreads) k_tab_fwd(const float* __restrict__ raw, int m, int G, PhiloxKey key,
                                                         uint32_t step, uint32_t rank, uint32_t stream,
                                                         float2* __restrict__ events, TabHist th) {
  extern __shared__ double tsm[];  // [2][G] tables, then [kTabThreads] scan scratch, then [2][bins+2] counts
  double* s_tot = tsm + 2 * G;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_tot + kTabThreads);
  const int hsz = th.hist ? th.bins + 2 : 0;
  for (int i = threadIdx.x; i < 2 * hsz; i += kTabThreads) s_hist[i] = 0;
  const int s = blockIdx.x;
  const double delta = 1.0 / (G - 1);
  for (int o = 0; o < 2; ++o) {
    const Wbc p = constrain_wbc(raw + 6 * (int64_t)s + 3 * o);
    double* F = tsm + o * G;
    for (int i = threadIdx.x; i < G; i += kTabThreads) node<false>(i * delta, p, &F[i], nullptr, nullptr, nullptr);
    __syncthreads();
    trapezoid_scan(F, G, delta, s_tot);
    const double inv = 1.0 / F[G - 1];
    for (int i = threadIdx.x; i < G; i += kTabThreads) F[i] *= inv;
    __syncthreads();
  }
  for (int j = threadIdx.x; j < m; j += kTabThreads) {
    const int64_t e = (int64_t)s * m + j;
    float xo[2];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      const double* F = tsm + o * G;
      const double u = event_u(key, step, rank, stream, e, o);
      const int i = find_cell(F, G, u);
      xo[o] = (float)(i * delta + (u - F[i]) / (F[i + 1] - F[i]) * delta);
    }
    events[e] = make_float2(xo[0], xo[1]);
    if (th.hist) {
      atomicAdd(&s_hist[hist_bin(xo[0], th.lo0, th.sc0, th.bins)], 1u);
      atomicAdd(&s_hist[hsz + hist_bin(xo[1], th.lo1, th.sc1, th.bins)], 1u);
    }
  }
  if (th.hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * hsz; i += kTabThreads)
      if (s_hist[i]) atomicAdd(&th.hist[i], s_hist[i]);
  }
}

__global__ void __launch_bounds__(kTabThreads) k_tab_bwd(const float* __restrict__ raw, int m, int G, PhiloxKey key,
                                                         uint32_t step, uint32_t rank, uint32_t stream,
                                                         const float2* __restrict__ dy, float* __restrict__ draw) {
  extern __shared__ double tsm[];  // [2 obs][4: F, dF/dw, dF/db, dF/dc][G], then scratch
  double* s_tot = tsm + 8 * G;
  const int s = blockIdx.x;
  const double delta = 1.0 / (G - 1);
  Wbc par[2];
  for (int o = 0; o < 2; ++o) {
    par[o] = constrain_wbc(raw + 6 * (int64_t)s + 3 * o);
    double* T = tsm + o * 4 * G;
    for (int i = threadIdx.x; i < G; i += kTabThreads)
      node<true>(i * delta, par[o], &T[i], &T[G + i], &T[2 * G + i], &T[3 * G + i]);
    __syncthreads();
    for (int q = 0; q < 4; ++q) trapezoid_scan(T + q * G, G, delta, s_tot);
    // F_i = S_i / S_end, dF_i = (dS_i S_end - S_i dS_end) / S_end^2 (quotient rule)
    const double S_end = T[G - 1], dW_end = T[2 * G - 1], dB_end = T[3 * G - 1], dC_end = T[4 * G - 1];
    __syncthreads();
    const double inv = 1.0 / S_end, inv2 = inv * inv;
    for (int i = threadIdx.x; i < G; i += kTabThreads) {
      const double S = T[i];
      T[i] = S * inv;
      T[G + i] = (T[G + i] * S_end - S * dW_end) * inv2;
      T[2 * G + i] = (T[2 * G + i] * S_end - S * dB_end) * inv2;
      T[3 * G + i] = (T[3 * G + i] * S_end - S * dC_end) * inv2;
    }
    __syncthreads();
  }
  double acc[6] = {0, 0, 0, 0, 0, 0};  // sum over this thread's events of dy * dx/dtheta
  for (int j = threadIdx.x; j < m; j += kTabThreads) {
    const int64_t e = (int64_t)s * m + j;
    const float2 g = dy[e];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      const double* T = tsm + o * 4 * G;
      const double u = event_u(key, step, rank, stream, e, o);
      const int i = find_cell(T, G, u);
      const double d = T[i + 1] - T[i], a = u - T[i];
      const double scale = -delta / (d * d) * (double)(o ? g.y : g.x);
#pragma unroll
      for (int q = 1; q <= 3; ++q) {
        const double* dF = T + q * G;
        acc[3 * o + q - 1] += scale * (dF[i] * d + a * (dF[i + 1] - dF[i]));
      }
    }
  }
  // fixed-order block reduction of the six sums
  for (int q = 0; q < 6; ++q) {
    s_tot[threadIdx.x] = acc[q];
    __syncthreads();
    for (int w = kTabThreads / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) s_tot[threadIdx.x] += s_tot[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const int o = q / 3, jj = q % 3;
      const float r = raw[6 * (int64_t)s + q];
      const double chain = jj == 0 ? par[o].w * (1.0 - par[o].w) : (r > 20.0f ? 1.0 : sigmoid_d((double)r));
      draw[6 * (int64_t)s + q] = (float)(s_tot[0] * chain);
    }
    __syncthreads();
  }
}

static size_t tab_smem(int G, bool bwd, int bins = 0) {
  return sizeof(double) * ((bwd ? 8 : 2) * (size_t)G + kTabThreads) + (bins > 0 ? sizeof(uint32_t) * 2 * (bins + 2) : 0);
}

bool tabulated_ok(int G) { return G >= 3 && G <= kTabMaxG; }

void launch_sample_tabulated(const float* raw, int k, int m, int G, uint64_t seed, uint32_t step, uint32_t rank,
                             uint32_t stream_id, float* events, cudaStream_t st, uint32_t* hist, int bins,
                             const float* lo, const float* hi) {
  TabHist th{nullptr, 0, 0.f, 0.f, 0.f, 0.f};
  if (hist && bins > 0) {
    th.hist = hist;
    th.bins = bins;
    th.lo0 = lo[0];
    th.lo1 = lo[1];
    th.sc0 = (float)bins / (hi[0] - lo[0]);  // fp32, as the quadratic sampler (R22)
    th.sc1 = (float)bins / (hi[1] - lo[1]);
  }
  const size_t sm = tab_smem(G, false, th.bins);
  static size_t configured = 0;
  if (sm > configured) {
    cudaFuncSetAttribute(k_tab_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = sm;
  }
  k_tab_fwd<<<k, kTabThreads, sm, st>>>(raw, m, G, make_key(seed), step, rank, stream_id,
                                         reinterpret_cast<float2*>(events), th);
  count_launch();
}

void launch_sample_tabulated_bwd(const float* raw, int k, int m, int G, uint64_t seed, uint32_t step, uint32_t rank,
                                 uint32_t stream_id, const float* dy, float* draw, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_tab_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab_smem(kTabMaxG, true));
    configured = true;
  }
  k_tab_bwd<<<k, kTabThreads, tab_smem(G, true), st>>>(raw, m, G, make_key(seed), step, rank, stream_id,
                                                        reinterpret_cast<const float2*>(dy), draw);
  count_launch();
}

}  // namespace sagips
