// mma_ts_rate.cu -- issue rate of the fused kernels' MMA phases on one SM:
// 8 K-steps x 3 products (bf16x3: Ah.Bh, Al.Bh, Ah.Bl) of M128 N128 K16, A from
// TMEM (TS) or from shared memory (SS), B from shared memory, issued by one
// converged warp (elect.sync), committed, waited; repeated.  Prints cycles
// per MMA.  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_00051_b200/csrc \
//        tests/tools/mma_ts_rate.cu -o /tmp/mma_ts_rate && /tmp/mma_ts_rate
#include <cstdio>

#include "tc_util.cuh"

using namespace sagips::tc;

__device__ __forceinline__ void mma_ts_warp(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// mode 0: TS bf16x3 forward (K-major B); 1: SS bf16x3; 2: TS 1 product; 3: SS 1 product;
// 4: TS bf16x3 with MN-major B (dgrad); 5: two accumulators alternating (TS, bf16x3)
__global__ void __launch_bounds__(128, 1) k_rate(int mode, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * 32768 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;  // bf16 1.0
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  const uint32_t bh = smem_u32(smem), bl = bh + 32768, sah = bh + 65536, sal = bh + 98304;
  if (warp == 0) {
    const bool mn = mode == 4;
    const uint32_t id = make_idesc_bf16(128, 128, 0, mn ? 1 : 0);
    const bool ts = (mode != 1 && mode != 3);
    const bool x3 = (mode != 2 && mode != 3);
    unsigned long long t0 = 0;
    for (int rep = 0; rep <= reps; ++rep) {
      if (rep == 1) t0 = clock64();
      const uint32_t acc = (mode == 5 && (rep & 1)) ? tm + 256 : tm;
      const uint32_t ah = acc + 128, al = acc + 192;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = mn ? k * 2048 : (k >> 2) * 16384 + (k & 3) * 32;
        const uint64_t dh = mn ? make_desc(bh + off, 16384, 1024) : make_desc(bh + off, 16, 1024);
        const uint64_t dl = mn ? make_desc(bl + off, 16384, 1024) : make_desc(bl + off, 16, 1024);
        const uint32_t ko = (k >> 2) * 16384 + (k & 3) * 32;
        if (ts) {
          mma_ts_warp(acc, ah + 8 * k, dh, id, k > 0);
          if (x3) {
            mma_ts_warp(acc, al + 8 * k, dh, id, 1);
            mma_ts_warp(acc, ah + 8 * k, dl, id, 1);
          }
        } else {
          mma_bf16_warp(acc, make_desc(sah + ko, 16, 1024), dh, id, k > 0);
          if (x3) {
            mma_bf16_warp(acc, make_desc(sal + ko, 16, 1024), dh, id, 1);
            mma_bf16_warp(acc, make_desc(sah + ko, 16, 1024), dl, id, 1);
          }
        }
      }
      if (mode != 5 || (rep & 1)) {
        mma_commit_warp(&bar);
        static_cast<void>(0);
      }
      if (mode != 5 || (rep & 1)) {
        // wait for this phase (as the fused kernels do between layers)
        const uint32_t ph = (mode == 5) ? ((rep >> 1) & 1) : (rep & 1);
        mbar_wait(&bar, ph);
      }
    }
    const unsigned long long t1 = clock64();
    if (tid == 0) out[mode] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 8);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 1024);
  const int reps = 400;
  const char* names[6] = {"TS bf16x3 K-major B", "SS bf16x3 K-major B", "TS 1 product", "SS 1 product",
                          "TS bf16x3 MN-major B", "TS bf16x3, 2 accumulators alternating"};
  for (int mode = 0; mode < 6; ++mode) {
    k_rate<<<1, 128, 4 * 32768 + 1024>>>(mode, reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    unsigned long long c;
    cudaMemcpy(&c, d + mode, 8, cudaMemcpyDeviceToHost);
    const int per = (mode == 2 || mode == 3) ? 8 : 24;
    printf("%-40s %7.1f cycles per MMA (%d per phase, commit + wait per phase)\n", names[mode],
           (double)c / ((double)reps * per), per);
  }
  return 0;
}
