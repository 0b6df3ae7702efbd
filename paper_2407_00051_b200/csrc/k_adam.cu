// k_adam.cu -- Adam (PyTorch form, R7) and the ascending fold of packets.
//
//   m <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2
//   p <- p - (lr / bc1) * m / (sqrt(v) / sqrt(bc2) + eps),  bc_i = 1 - b_i^tau
// bc1 / sqrt(bc2) are computed on the host in double, as torch.optim.Adam.
#include "internal.h"

namespace sagips {

__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, float step_size, float bc2_sqrt, float b1, float b2,
                       float eps) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float pi = p[i], mi = m[i], vi = v[i];
    adam_elem(pi, g[i], mi, vi, step_size, bc2_sqrt, b1, b2, eps);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
  }
}

void launch_adam(float* p, const float* g, float* m, float* v, int64_t n, double lr, int64_t tau, double b1,
                 double b2, double eps, cudaStream_t st) {
  if (n <= 0) return;
  const double bc1 = 1.0 - std::pow(b1, (double)tau);
  const double bc2 = 1.0 - std::pow(b2, (double)tau);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
  k_adam<<<blocks, 256, 0, st>>>(p, g, m, v, n, (float)(lr / bc1), (float)std::sqrt(bc2), (float)b1, (float)b2,
                                 (float)eps);
  count_launch();
}

// Fused gradient reduction + Adam for the discriminator (one launch per D
// step): each segment is one parameter tensor whose gradient arrives as
// per-CTA partials; block = 32 elements x 8 part groups (group g sums parts
// g, g+8, ... in order, the 8 group sums are added in order -- deterministic),
// then the element's Adam update (the same arithmetic as k_adam).
__global__ void __launch_bounds__(256) k_reduce_adam(const __grid_constant__ RedAdamArgs a) {
  __shared__ float red[8][33];
  int si = 0;
  while (si + 1 < a.nseg && (int)blockIdx.x >= a.seg[si + 1].block0) ++si;
  const RedSeg& sg = a.seg[si];
  const int jl = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int j = (blockIdx.x - sg.block0) * 32 + jl;
  float s = 0.f;
  if (j < sg.n) {
#pragma unroll 4
    for (int p = grp; p < sg.nparts; p += 8) s += __ldg(sg.part + (int64_t)p * sg.ld + j);
  }
  red[grp][jl] = s;
  __syncthreads();
  if (grp == 0 && j < sg.n) {
    float gi = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) gi += red[k][jl];
    sg.g[j] = gi;
    if (a.adam) {
      float pj = sg.p[j], mj = sg.m[j], vj = sg.v[j];
      adam_elem(pj, gi, mj, vj, a.step_size, a.bc2_sqrt, a.b1, a.b2, a.eps);
      sg.p[j] = pj;
      sg.m[j] = mj;
      sg.v[j] = vj;
    }
  }
}

void launch_reduce_adam(RedAdamArgs& a, double lr, int64_t tau, double b1, double b2, double eps, cudaStream_t st) {
  int blocks = 0;
  for (int i = 0; i < a.nseg; ++i) {
    a.seg[i].block0 = blocks;
    blocks += (a.seg[i].n + 31) / 32;
  }
  const double bc1 = 1.0 - std::pow(b1, (double)tau);
  const double bc2 = 1.0 - std::pow(b2, (double)tau);
  a.step_size = (float)(lr / bc1);
  a.bc2_sqrt = (float)std::sqrt(bc2);
  a.b1 = (float)b1;
  a.b2 = (float)b2;
  a.eps = (float)eps;
  k_reduce_adam<<<blocks, 256, 0, st>>>(a);
  count_launch();
}

// out[i] = (((P_0[i] + P_1[i]) + P_2[i]) + ...)  / divisor over the given
// packets in the given (ascending origin) order (R10).  Pointers may be
// local or peer-mapped (NVLink) addresses.
__global__ void k_fold(PacketList pl, int64_t n, float* __restrict__ out, float divisor) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = pl.p[0][i];
    for (int j = 1; j < pl.count; ++j) acc += pl.p[j][i];
    out[i] = acc / divisor;
  }
}

void launch_fold(const PacketList& pl, int64_t n, float* out, float divisor, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 2);
  k_fold<<<blocks, 256, 0, st>>>(pl, n, out, divisor);
  count_launch();
}

}  // namespace sagips
