// tmem_a_check.cu -- standalone check of the tcgen05.mma form with the A
// operand in tensor memory (kind::f16, M = 128, N = 128, K = 128 in 8 steps),
// as the fused discriminator kernels use it: row m of A lives in TMEM lane m,
// K element k of that row in 32-bit column k / 2 (low half = even k); B is a
// shared-memory SW128 operand, K-major (D = A B^T, the forward) or MN-major
// (D = A B, the dgrad).  Also times back-to-back MMAs with A from TMEM vs A
// from shared memory.  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_00051_b200/csrc \
//        tests/tools/tmem_a_check.cu -o /tmp/tmem_a_check && /tmp/tmem_a_check
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_util.cuh"

using namespace sagips::tc;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// A [128][128] bf16 bits, B [128][128] bf16 bits (row-major [r][c]); D out [128][128] fp32
__global__ void __launch_bounds__(128, 1) k_check(const uint16_t* A, const uint16_t* B, float* D, int mn_major,
                                                  int reps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem;              // 32 KiB SW128 tile
  uint8_t* sA = smem + 32768;      // 32 KiB SW128 tile (timing reference: A from smem)
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 128; i += 128) {
    const int r = i >> 7, c = i & 127;
    *reinterpret_cast<uint16_t*>(sB + sw128_offset(r, c, 128)) = B[i];
    *reinterpret_cast<uint16_t*>(sA + sw128_offset(r, c, 128)) = A[i];
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t accd = tm, areg = tm + 128;
  // A row (32 warp + lane) -> TMEM lane, columns areg .. areg + 63 (2 bf16 per column)
  {
    const int row = tid;
    uint32_t w[32];
    for (int half = 0; half < 2; ++half) {
      for (int j = 0; j < 32; ++j) {
        const int k = 64 * half + 2 * j;
        w[j] = (uint32_t)A[row * 128 + k] | ((uint32_t)A[row * 128 + k + 1] << 16);
      }
      tmem_st32(areg + ((uint32_t)(32 * warp) << 16) + 32 * half, w);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t idesc = make_idesc_bf16(128, 128, 0, mn_major);
  const uint32_t bb = smem_u32(sB), ab = smem_u32(sA);
  unsigned long long t0 = 0, t1 = 0, t2 = 0;
  if (tid == 0) {
    for (int rep = 0; rep < 1 + 2 * reps; ++rep) {
      if (rep == 1) t0 = clock64();
      if (rep == 1 + reps) t1 = clock64();
      const bool from_smem = rep > reps;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bd = mn_major ? make_desc(bb + k * 2048, 16384, 1024)
                                     : make_desc(bb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
        if (from_smem)
          mma_bf16(accd, make_desc(ab + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), bd, idesc, k > 0);
        else
          mma_ts(accd, areg + 8 * k, bd, idesc, k > 0);
      }
      if (rep == 0 || rep == reps || rep == 2 * reps) {
        mma_commit(&bar);
        mbar_wait(&bar, (rep == 0) ? 0 : (rep == reps ? 1 : 0));
        if (rep == 2 * reps) t2 = clock64();
      }
    }
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
  __syncthreads();
  tc_fence_after();
  // the last group of reps was A from smem (same values): D is A B^T (or A B) either way
  float v[32];
  for (int c0 = 0; c0 < 128; c0 += 32) {
    tmem_ld32(accd + ((uint32_t)(32 * warp) << 16) + c0, v);
    for (int j = 0; j < 32; ++j) D[tid * 128 + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tm);
}

// the same with a single rep of A from TMEM only, to check its values
__global__ void __launch_bounds__(128, 1) k_check_ts(const uint16_t* A, const uint16_t* B, float* D, int mn_major) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 128; i += 128) {
    const int r = i >> 7, c = i & 127;
    *reinterpret_cast<uint16_t*>(sB + sw128_offset(r, c, 128)) = B[i];
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base, accd = tm, areg = tm + 128;
  uint32_t w[32];
  for (int half = 0; half < 2; ++half) {
    for (int j = 0; j < 32; ++j) {
      const int k = 64 * half + 2 * j;
      w[j] = (uint32_t)A[tid * 128 + k] | ((uint32_t)A[tid * 128 + k + 1] << 16);
    }
    tmem_st32(areg + ((uint32_t)(32 * warp) << 16) + 32 * half, w);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = make_idesc_bf16(128, 128, 0, mn_major);
    const uint32_t bb = smem_u32(sB);
    for (int k = 0; k < 8; ++k) {
      const uint64_t bd = mn_major ? make_desc(bb + k * 2048, 16384, 1024)
                                   : make_desc(bb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      mma_ts(accd, areg + 8 * k, bd, idesc, k > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  float v[32];
  for (int c0 = 0; c0 < 128; c0 += 32) {
    tmem_ld32(accd + ((uint32_t)(32 * warp) << 16) + c0, v);
    for (int j = 0; j < 32; ++j) D[tid * 128 + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tm);
}

static uint16_t bf16_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float bf16_val(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

int main() {
  const int n = 128 * 128;
  std::vector<uint16_t> A(n), B(n);
  srand(7);
  for (int i = 0; i < n; ++i) {
    A[i] = bf16_bits((rand() / (float)RAND_MAX - 0.5f) * 2.f);
    B[i] = bf16_bits((rand() / (float)RAND_MAX - 0.5f) * 2.f);
  }
  uint16_t *dA, *dB;
  float* dD;
  unsigned long long* dc;
  cudaMalloc(&dA, 2 * n);
  cudaMalloc(&dB, 2 * n);
  cudaMalloc(&dD, 4 * n);
  cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), 2 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 2 * n, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  cudaFuncSetAttribute(k_check_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  int bad_total = 0;
  for (int mn = 0; mn < 2; ++mn) {
    k_check_ts<<<1, 128, 32768 + 1024>>>(dA, dB, dD, mn);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("kernel error: %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> D(n);
    cudaMemcpy(D.data(), dD, 4 * n, cudaMemcpyDeviceToHost);
    int bad = 0;
    double worst = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 128; ++c) {
        double ref = 0;
        for (int k = 0; k < 128; ++k)
          ref += (double)bf16_val(A[r * 128 + k]) * (mn ? bf16_val(B[k * 128 + c]) : bf16_val(B[c * 128 + k]));
        const double err = std::abs(D[r * 128 + c] - ref);
        worst = std::max(worst, err);
        if (err > 1e-4 * (1 + std::abs(ref))) ++bad;
      }
    printf("A from TMEM, B %s: %d bad of %d, max abs err %.3g\n", mn ? "MN-major (D = A B)" : "K-major (D = A B^T)",
           bad, n, worst);
    bad_total += bad;
  }
  const int reps = 2000;
  k_check<<<1, 128, 65536 + 1024>>>(dA, dB, dD, 0, reps, dc);
  cudaDeviceSynchronize();
  unsigned long long cyc[2];
  cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
  printf("cycles per M128 N128 K16 MMA (single thread issue): A from TMEM %.1f, A from smem %.1f\n",
         cyc[0] / (8.0 * reps), cyc[1] / (8.0 * reps));
  printf(bad_total == 0 ? "TMEM_A_OK\n" : "TMEM_A_FAIL\n");
  return bad_total != 0;
}
