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

// Ten rounds; mulhi/mullo map to IMAD.WIDE on sm_100a.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, PhiloxKey key) {
  uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint4 philox_call(PhiloxKey key, uint32_t index, uint32_t step,
                                             uint32_t rank, uint32_t stream) {
  return philox4x32_10(make_uint4(index, step, rank, stream), key);
}

__device__ __forceinline__ uint32_t word_of(uint4 r, int lane) {
  return lane == 0 ? r.x : lane == 1 ? r.y : lane == 2 ? r.z : r.w;
}

// u = (2 * (w >> 9) + 1) * 2^-24 in (0, 1), exact in fp32 (R-UNIF).
__device__ __forceinline__ float uniform_open01(uint32_t w) {
  return __uint2float_rn(2u * (w >> 9) + 1u) * 5.9604644775390625e-8f;
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

// histogram bin: 0 underflow/NaN, 1..bins, bins+1 overflow.
__device__ __forceinline__ int hist_bin(float y, float lo, float scale, int bins) {
  const float t = __fmul_rn(__fsub_rn(y, lo), scale);
  if (!(t >= 0.0f)) return 0;
  if (t >= static_cast<float>(bins)) return bins + 1;
  return static_cast<int>(t) + 1;
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

}  // namespace sagips
