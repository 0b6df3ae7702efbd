// common.cuh -- shared device helpers of libsagips (sm_100a).
//
// Philox4x32-10 (Salmon et al., SC'11) with the counter layout of DESIGN.md
// R-RNG: key = (seed lo, seed hi), ctr = (index, step, rank, stream), and the
// word stream numbering "word i = word (i % 4) of call i / 4".  This is the
// device implementation; the oracle has its own, independent one.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sagips {

enum Stream : uint32_t {
  kStreamRef = 0, kStreamShard = 1, kStreamInitG = 2, kStreamInitD = 3,
  kStreamNoise = 4, kStreamFake = 5, kStreamReal = 6
};

struct PhiloxKey { uint32_t k0, k1; };

__host__ __device__ inline PhiloxKey make_key(uint64_t seed) {
  return PhiloxKey{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)};
}

// Ten rounds.  Each 32x32 -> 64-bit product is one IMAD.WIDE.U32 (hi and lo
// together); the key bumps k + r*W are compile-time-unrolled adds that the
// compiler hoists out of grid-stride loops.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, PhiloxKey key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t k0 = key.k0 + (uint32_t)r * 0x9E3779B9u;
    const uint32_t k1 = key.k1 + (uint32_t)r * 0xBB67AE85u;
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0);
  }
  return c;
}

__device__ __forceinline__ uint4 philox_call(PhiloxKey key, uint32_t index, uint32_t step,
                                             uint32_t rank, uint32_t stream) {
  return philox4x32_10(make_uint4(index, step, rank, stream), key);
}

// The ten round keys, computed once per thread (a grid-stride loop calling
// philox4x32_10 recomputes k + r*W every call).
struct PhiloxRoundKeys {
  uint32_t k0[10], k1[10];
};
__device__ __forceinline__ PhiloxRoundKeys round_keys(PhiloxKey key) {
  PhiloxRoundKeys rk;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    rk.k0[r] = key.k0 + (uint32_t)r * 0x9E3779B9u;
    rk.k1[r] = key.k1 + (uint32_t)r * 0xBB67AE85u;
  }
  return rk;
}
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const PhiloxRoundKeys& rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ rk.k0[r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ rk.k1[r],
                   (uint32_t)p0);
  }
  return c;
}

__device__ __forceinline__ uint32_t word_of(uint4 r, int lane) {
  return lane == 0 ? r.x : lane == 1 ? r.y : lane == 2 ? r.z : r.w;
}

// u = (2 * (w >> 9) + 1) * 2^-24 in (0, 1), exact in fp32 (R-UNIF), built
// from the bits: 1 + (w >> 9) 2^-23 is the float 0x3F800000 | (w >> 9), and
// subtracting (1 - 2^-24) leaves (2 (w >> 9) + 1) 2^-24, which has <= 24
// significant bits, so the one rounded subtraction is exact.
__device__ __forceinline__ float uniform_open01(uint32_t w) {
  const float one_m = __uint_as_float(0x3F800000u | (w >> 9));
  return __fsub_rn(one_m, 0.99999994039535522461f);
}

// Lemire multiply-shift (R-BOOT): (w * n) >> 32.
__device__ __forceinline__ uint32_t lemire(uint32_t w, uint32_t n) {
  return static_cast<uint32_t>((static_cast<uint64_t>(w) * n) >> 32);
}

// Q(u; c) = c0 + u * (c1 + u * c2), every operation rounded (no FMA), so
// that histogram bins are a deterministic function of (c, u) (R22).
__device__ __forceinline__ float quantile_f32(float u, float c0, float c1, float c2) {
  const float a = __fmul_rn(u, c2);
  const float b = __fadd_rn(c1, a);
  const float d = __fmul_rn(u, b);
  return __fadd_rn(c0, d);
}

// histogram bin: 0 underflow/NaN, 1..bins, bins+1 overflow.  t = (y-lo)*scale
// in fp32 (two roundings, as R22); clamping t to [-1, bins] (fmaxf drops a
// NaN) and flooring gives -1 for t < 0 or NaN, bins for t >= bins.
// floor(t) for t in [-1, bins] (bins <= 4096) without the quarter-rate F2I:
// t + 1.5 * 2^23 rounded down is exactly 1.5 * 2^23 + floor(t) (unit ulp
// there), whose bits are 0x4B400000 + floor(t).
__device__ __forceinline__ int hist_bin(float y, float lo, float scale, int bins) {
  const float t = __fmul_rn(__fsub_rn(y, lo), scale);
  const float c = fminf(fmaxf(t, -1.0f), static_cast<float>(bins));
  return __float_as_int(__fadd_rd(c, 12582912.0f)) - 0x4B400000 + 1;
}

__device__ __forceinline__ float softplus_f(float x) {
  return x > 20.0f ? x : log1pf(expf(x));
}
__device__ __forceinline__ float sigmoid_f(float x) {
  return 1.0f / (1.0f + expf(-x));
}
__device__ __forceinline__ float softplus_grad_f(float x) {
  return x > 20.0f ? 1.0f : sigmoid_f(x);
}
// log(1 + e^-|z|) + max(-z, 0) = softplus(-z)
__device__ __forceinline__ float softplus_neg(float z) {
  return fmaxf(-z, 0.0f) + log1pf(expf(-fabsf(z)));
}

// loss = scale * sum of part[0 .. nparts) in ascending order, by one block:
// up to kLossCap partials are loaded by the whole block at once (one round
// trip) into sp, then summed by thread 0; writes the stats' loss and the
// non-finite flag (the SPEC's NaN guard).  k_finish_loss, and the extra
// block of the kernels that absorb it (k_reduce_adam, k_sample_bwd).
constexpr int kLossCap = 512;
__device__ inline void finish_loss_block(const double* part, int nparts, double scale, float* out, uint32_t* nonfinite,
                                         double* sp) {
  for (int p = threadIdx.x; p < nparts && p < kLossCap; p += blockDim.x) sp[p] = part[p];
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int p = 0; p < nparts; ++p) v += p < kLossCap ? sp[p] : part[p];
    const float l = (float)(v * scale);
    *out = l;
    if (!isfinite(l)) *nonfinite = 1u;
  }
}

}  // namespace sagips
