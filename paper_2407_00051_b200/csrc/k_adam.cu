// k_adam.cu -- Adam (PyTorch form, R7) and the ascending fold of packets.
//
//   m <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2
//   p <- p - (lr / bc1) * m / (sqrt(v) / sqrt(bc2) + eps),  bc_i = 1 - b_i^tau
// bc1 / sqrt(bc2) are computed on the host in double, as torch.optim.Adam.
#include "internal.h"

namespace sagips {

__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, float step_size, float bc2_sqrt, float b1, float b2,
                       float eps, int vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nq = vec ? n >> 2 : 0;  // quads when every array is 16-byte aligned (same per-element arithmetic)
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += stride) {
    float4 pi = reinterpret_cast<const float4*>(p)[q], mi = reinterpret_cast<const float4*>(m)[q],
           vi = reinterpret_cast<const float4*>(v)[q];
    const float4 gi = reinterpret_cast<const float4*>(g)[q];
    adam_elem(pi.x, gi.x, mi.x, vi.x, step_size, bc2_sqrt, b1, b2, eps);
    adam_elem(pi.y, gi.y, mi.y, vi.y, step_size, bc2_sqrt, b1, b2, eps);
    adam_elem(pi.z, gi.z, mi.z, vi.z, step_size, bc2_sqrt, b1, b2, eps);
    adam_elem(pi.w, gi.w, mi.w, vi.w, step_size, bc2_sqrt, b1, b2, eps);
    reinterpret_cast<float4*>(p)[q] = pi;
    reinterpret_cast<float4*>(m)[q] = mi;
    reinterpret_cast<float4*>(v)[q] = vi;
  }
  for (int64_t i = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
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
  auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  const int vec = (a16(p) && a16(g) && a16(m) && a16(v) && n >= (int64_t(1) << 20)) ? 1 : 0;  // large only
  const int blocks = (int)std::min<int64_t>((n / (vec ? 4 : 1) + 255) / 256, 148 * 8);
  k_adam<<<blocks, 256, 0, st>>>(p, g, m, v, n, (float)(lr / bc1), (float)std::sqrt(bc2), (float)b1, (float)b2,
                                 (float)eps, vec);
  count_launch();
}

// Fused gradient reduction + Adam for the discriminator (one launch per D
// step): each segment is one parameter tensor whose gradient arrives as
// per-CTA partials; block = 32 elements x 8 part groups (group g sums parts
// g, g+8, ... in order, the 8 group sums are added in order -- deterministic),
// then the element's Adam update (the same arithmetic as k_adam).
__global__ void __launch_bounds__(256) k_reduce_adam(const __grid_constant__ RedAdamArgs a) {
  __shared__ float red[8][33];
  if (a.loss_part && blockIdx.x == gridDim.x - 1) {  // the extra block: the step's D loss
    __shared__ double sp[kLossCap];
    finish_loss_block(a.loss_part, a.loss_nparts, a.loss_scale, a.loss_out, a.nonfinite, sp);
    return;
  }
  int si = 0;
  while (si + 1 < a.nseg && (int)blockIdx.x >= a.seg[si + 1].block0) ++si;
  const RedSeg& sg = a.seg[si];
  const int jl = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int j = (blockIdx.x - sg.block0) * 32 + jl;
  float s = 0.f;
  if (j < sg.n) {
#pragma unroll 8  // (more loads in flight; the sum order is unchanged)
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
  if (a.loss_part) ++blocks;  // + the loss block
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
