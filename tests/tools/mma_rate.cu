// Isolated tcgen05 MMA-rate microbenchmark (diagnostic tool, not the product):
// one CTA per SM issues the per-tile MMA sequences of the layer passes on
// operands resident in shared memory (garbage data) and reports cycles per
// tile.  Shows whether the layer kernels' per-tile period is set by the MMA
// pipe itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_00051_b200/csrc \
//        tests/tools/mma_rate.cu -o /tmp/mma_rate && /tmp/mma_rate
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_util.cuh"

using namespace sagips::tc;

constexpr uint32_t kPlane = 128 * 128 * 2;

// mode 0: forward (3 products x 8 K-steps, one accumulator)
// mode 1: wgrad/dgrad backward (wgrad hi: 8 x (W, db); dgrad hi: 16; wgrad lo: 8 x (W, db); dgrad lo: 8)
// mode 2: as 1 without the db MMAs
// mode 3: forward, M128 N256 (two 128-column accumulators' worth per MMA), 12 MMAs per tile (same FLOPs)
__global__ void __launch_bounds__(128, 1) k_rate(int mode, int tiles, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * kPlane + 512);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(slot);
  for (int i = threadIdx.x; i < 128; i += blockDim.x) reinterpret_cast<uint32_t*>(smem + 4 * kPlane)[i] = 0x3F803F80u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + kPlane, c = b + kPlane, w = c + kPlane;
    const uint64_t ones = make_desc(smem_u32(smem + 4 * kPlane), 128, 256, 0);
    constexpr uint32_t id = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t id_w = make_idesc_bf16(128, 128, 1, 1);
    constexpr uint32_t id_d = make_idesc_bf16(128, 128, 0, 1);
    constexpr uint32_t id_b = make_idesc_bf16(128, 16, 1, 0);
    constexpr uint32_t id256 = make_idesc_bf16(128, 256, 0, 0);
    const uint32_t acc_w = tmem + 256, acc_b = tmem + 384;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (uint32_t)((t & 1) * 128);
      if (mode == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          mma_bf16(d, make_desc(b + off, 16, 1024), make_desc(w + off, 16, 1024), id, k > 0);
          mma_bf16(d, make_desc(a + off, 16, 1024), make_desc(w + off, 16, 1024), id, 1);
          mma_bf16(d, make_desc(a + off, 16, 1024), make_desc(c + off, 16, 1024), id, 1);
        }
      } else if (mode == 3) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // K = 64 per "tile" at N = 256: same FLOPs as mode 0
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          mma_bf16(tmem, make_desc(a + off, 16, 1024), make_desc(w + off, 16, 1024), id256, k > 0);
          mma_bf16(tmem, make_desc(b + off, 16, 1024), make_desc(w + off, 16, 1024), id256, 1);
          mma_bf16(tmem, make_desc(a + off, 16, 1024), make_desc(c + off, 16, 1024), id256, 1);
        }
      } else {
        const bool db = mode == 1;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048;
          const uint64_t g = make_desc(a + km, 16384, 1024);
          mma_bf16(acc_w, g, make_desc(b + km, 16384, 1024), id_w, 1);
          if (db) mma_bf16(acc_b, g, ones, id_b, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          const uint64_t g = make_desc(a + kk, 16, 1024);
          mma_bf16(d, g, make_desc(w + km, 16384, 1024), id_d, k > 0);
          mma_bf16(d, g, make_desc(c + km, 16384, 1024), id_d, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048;
          const uint64_t g = make_desc(c + km, 16384, 1024);
          mma_bf16(acc_w, g, make_desc(b + km, 16384, 1024), id_w, 1);
          if (db) mma_bf16(acc_b, g, ones, id_b, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          mma_bf16(d, make_desc(c + kk, 16, 1024), make_desc(w + km, 16384, 1024), id_d, 1);
        }
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const size_t sm = 4 * kPlane + 512 + 64;
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  unsigned long long* d_out;
  cudaMalloc(&d_out, sizeof(unsigned long long) * sms);
  unsigned long long h[256];
  const char* names[4] = {"fwd 3x8 M128N128K16", "bwd 40 N128 + 16 db(N16)", "bwd 40 N128 (no db)", "fwd as 12 M128N256K16"};
  const double flops[4] = {24, 40, 40, 24};  // M128N128K16-equivalents per tile
  for (int mode = 0; mode < 4; ++mode) {
    const int tiles = 400;
    k_rate<<<sms, 128, sm>>>(mode, tiles, d_out);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate<<<sms, 128, sm>>>(mode, tiles, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, d_out, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += (double)h[i];
    cyc /= sms;
    const double tf = flops[mode] * 2.0 * 128 * 128 * 16 * tiles * sms / (ms * 1e-3) / 1e12;
    printf("%-28s %7.0f cycles/tile (%5.1f per N128-MMA-equivalent), %.3f us/tile wall, %6.0f TFLOP/s  [%s]\n",
           names[mode], cyc / tiles, cyc / tiles / flops[mode], ms * 1e3 / tiles, tf,
           cudaGetErrorString(cudaGetLastError()));
  }
  printf("(SM clock attribute %d MHz)\n", clk / 1000);
  return 0;
}
