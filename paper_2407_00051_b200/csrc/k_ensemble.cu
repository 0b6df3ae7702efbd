// k_ensemble.cu -- ensemble response and normalised residuals (§8(f) rows 2
// and 4): Eq. 7 p_hat = (1/M) sum_i G_i(n), Eq. 8 sigma = sqrt((1/M) sum_i
// (G_i(n) - p_hat)^2), both averaged over the k noise vectors
// (P:332), and Eq. 6 r_hat = (p - p_hat) / p.
//
// One block per parameter j; thread t takes noise vectors t, t + 256, ...;
// sums in fp64 in a fixed order (members ascending, then a fixed tree over
// the threads), so the result is deterministic.
#include "ctx.h"

namespace sagips {

namespace {
constexpr int kEnsThreads = 256;
}

struct EnsTruth {
  double p[kEnsMaxParams];
  int have;
};

__global__ void __launch_bounds__(kEnsThreads) k_ensemble_stats(const float* __restrict__ preds, int M, int k, int P,
                                                                EnsTruth truth, double* __restrict__ out) {
  __shared__ double s_mean[kEnsThreads], s_std[kEnsThreads];
  const int j = blockIdx.x, t = threadIdx.x;
  double sm = 0.0, ss = 0.0;
  for (int s = t; s < k; s += kEnsThreads) {
    double mean = 0.0;
    for (int i = 0; i < M; ++i) mean += (double)preds[((int64_t)i * k + s) * P + j];
    mean /= M;  // Eq. 7
    double var = 0.0;
    for (int i = 0; i < M; ++i) {
      const double d = (double)preds[((int64_t)i * k + s) * P + j] - mean;
      var += d * d;
    }
    sm += mean;
    ss += sqrt(var / M);  // Eq. 8
  }
  s_mean[t] = sm;
  s_std[t] = ss;
  __syncthreads();
  for (int w = kEnsThreads / 2; w > 0; w >>= 1) {
    if (t < w) {
      s_mean[t] += s_mean[t + w];
      s_std[t] += s_std[t + w];
    }
    __syncthreads();
  }
  if (t == 0) {
    const double p_hat = s_mean[0] / k, sigma = s_std[0] / k;  // batch averages
    out[j] = p_hat;
    out[P + j] = sigma;
    out[2 * P + j] = truth.have ? (truth.p[j] - p_hat) / truth.p[j] : __longlong_as_double(0x7ff8000000000000ll);
  }
}

int launch_ensemble_stats(const float* preds, int M, int k, int P, const double* p_true, double* out_dev,
                          cudaStream_t st) {
  EnsTruth truth{};
  truth.have = p_true != nullptr;
  for (int j = 0; j < P && p_true; ++j) truth.p[j] = p_true[j];
  k_ensemble_stats<<<P, kEnsThreads, 0, st>>>(preds, M, k, P, truth, out_dev);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace sagips
