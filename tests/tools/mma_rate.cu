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
#define MMA(...) (kWarp ? mma_bf16_warp(__VA_ARGS__) : mma_bf16(__VA_ARGS__))

constexpr uint32_t kPlane = 128 * 128 * 2;

// mode 0: forward (3 products x 8 K-steps, one accumulator)
// mode 1: wgrad/dgrad backward (wgrad hi: 8 x (W, db); dgrad hi: 16; wgrad lo: 8 x (W, db); dgrad lo: 8)
// mode 2: as 1 without the db MMAs
// mode 3: forward, M128 N256 (two 128-column accumulators' worth per MMA), 12 MMAs per tile (same FLOPs)
// modes 4-7: 24 MMAs of one operand-major combination; mode 8: the kT (transposed dgrad) backward
template <bool kWarp>
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
  if (kWarp ? warp == 0 : threadIdx.x == 0) {
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
          MMA(d, make_desc(b + off, 16, 1024), make_desc(w + off, 16, 1024), id, k > 0);
          MMA(d, make_desc(a + off, 16, 1024), make_desc(w + off, 16, 1024), id, 1);
          MMA(d, make_desc(a + off, 16, 1024), make_desc(c + off, 16, 1024), id, 1);
        }
      } else if (mode >= 4 && mode <= 7) {
        // 24 M128N128K16 MMAs of one operand layout: 4 wgrad (A, B MN-major),
        // 5 dgrad (A K-major, B MN-major), 6 dgrad-T (A MN-major, B K-major), 7 fwd (both K-major)
        const uint32_t idm = mode == 4 ? id_w : mode == 5 ? id_d : mode == 6 ? make_idesc_bf16(128, 128, 1, 0) : id;
        const bool amn = mode == 4 || mode == 6, bmn = mode == 4 || mode == 5;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
            const uint64_t ad = amn ? make_desc(a + km, 16384, 1024) : make_desc(a + kk, 16, 1024);
            const uint64_t bd = bmn ? make_desc(w + km, 16384, 1024) : make_desc(w + kk, 16, 1024);
            MMA(d, ad, bd, idm, (r | k) ? 1u : 0u);
          }
      } else if (mode == 8) {  // the kT backward: wgrad hi + db, dgrad-T hi (2), wgrad lo + db, dgrad-T lo
        constexpr uint32_t id_dT = make_idesc_bf16(128, 128, 1, 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048;
          const uint64_t g = make_desc(a + km, 16384, 1024);
          MMA(acc_w, g, make_desc(b + km, 16384, 1024), id_w, 1);
          MMA(acc_b, g, ones, id_b, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          const uint64_t g = make_desc(a + kk, 16, 1024);
          MMA(d, make_desc(w + km, 16384, 1024), g, id_dT, k > 0);
          MMA(d, make_desc(c + km, 16384, 1024), g, id_dT, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048;
          const uint64_t g = make_desc(c + km, 16384, 1024);
          MMA(acc_w, g, make_desc(b + km, 16384, 1024), id_w, 1);
          MMA(acc_b, g, ones, id_b, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          MMA(d, make_desc(w + km, 16384, 1024), make_desc(c + kk, 16, 1024), id_dT, 1);
        }
      } else if (mode == 3) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // K = 64 per "tile" at N = 256: same FLOPs as mode 0
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          MMA(tmem, make_desc(a + off, 16, 1024), make_desc(w + off, 16, 1024), id256, k > 0);
          MMA(tmem, make_desc(b + off, 16, 1024), make_desc(w + off, 16, 1024), id256, 1);
          MMA(tmem, make_desc(a + off, 16, 1024), make_desc(c + off, 16, 1024), id256, 1);
        }
      } else {
        const bool db = mode == 1;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048;
          const uint64_t g = make_desc(a + km, 16384, 1024);
          MMA(acc_w, g, make_desc(b + km, 16384, 1024), id_w, 1);
          if (db) MMA(acc_b, g, ones, id_b, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          const uint64_t g = make_desc(a + kk, 16, 1024);
          MMA(d, g, make_desc(w + km, 16384, 1024), id_d, k > 0);
          MMA(d, g, make_desc(c + km, 16384, 1024), id_d, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t km = k * 2048;
          const uint64_t g = make_desc(c + km, 16384, 1024);
          MMA(acc_w, g, make_desc(b + km, 16384, 1024), id_w, 1);
          if (db) MMA(acc_b, g, ones, id_b, 1);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t kk = (k >> 2) * 16384 + (k & 3) * 32, km = k * 2048;
          MMA(d, make_desc(c + kk, 16, 1024), make_desc(w + km, 16384, 1024), id_d, 1);
        }
      }
    }
    if (kWarp) mma_commit_warp(bar); else mma_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
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
  cudaFuncSetAttribute(k_rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k_rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  unsigned long long* d_out;
  cudaMalloc(&d_out, sizeof(unsigned long long) * sms);
  unsigned long long h[256];
  const char* names[9] = {"fwd 3x8 M128N128K16", "bwd 40 N128 + 16 db(N16)", "bwd 40 N128 (no db)",
                          "fwd as 12 M128N256K16", "24 wgrad (A,B MN-major)", "24 dgrad (B MN-major)",
                          "24 dgrad-T (A MN-major)", "24 fwd (K-major)", "kT bwd 40 + 16 db"};
  const double flops[9] = {24, 40, 40, 24, 24, 24, 24, 24, 40};  // M128N128K16-equivalents per tile
  for (int wv = 0; wv < 2; ++wv)
  for (int mode = 0; mode < 9; ++mode) {
    auto kern = wv ? k_rate<true> : k_rate<false>;
    const int tiles = 400;
    kern<<<sms, 128, sm>>>(mode, tiles, d_out);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<sms, 128, sm>>>(mode, tiles, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, d_out, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += (double)h[i];
    cyc /= sms;
    const double tf = flops[mode] * 2.0 * 128 * 128 * 16 * tiles * sms / (ms * 1e-3) / 1e12;
    printf("%s %-28s %7.0f cycles/tile (%5.1f per N128-MMA-equivalent), %.3f us/tile wall, %6.0f TFLOP/s  [%s]\n",
           wv ? "warp  " : "thread", names[mode], cyc / tiles, cyc / tiles / flops[mode], ms * 1e3 / tiles, tf,
           cudaGetErrorString(cudaGetLastError()));
  }
  printf("(SM clock attribute %d MHz)\n", clk / 1000);
  return 0;
}
