// Microbenchmark: tcgen05.mma (kind::f16, bf16 -> fp32, SS mode, K-major
// operands) issue throughput per SM for M=128, several N, SWIZZLE_NONE vs
// SWIZZLE_128B operand layouts, and 1/2/4 independent accumulators issued
// round-robin (a single accumulator serialises on the D read-modify-write).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_bench tools/umma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1703_02529_b200/csrc/common.cuh"

using namespace ns;

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO = 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

NS_DEV void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

template <int N, int NACC, bool SW, int SBO = 128, int HAMMER = 0, int OFF = 0, int M = 128, int CE = 0, int TS = 0>
__global__ void __launch_bounds__(512, 1) mma_loop(int iters, int ksteps, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* A = smem;                      // 128 rows x 128 B per 4 K-steps (sw) / 4 KB per step
  uint8_t* B = smem + 32768;
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (32768 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (HAMMER && threadIdx.x >= 32) {
    // CUDA-core shared-memory traffic concurrent with the MMAs (LDS.128 + STS.128)
    uint4* buf = reinterpret_cast<uint4*>(smem + 65536);
    uint4 acc = make_uint4(0, 0, 0, 0);
    int i = threadIdx.x - 32;
    while (!stop) {
      for (int r = 0; r < 64; ++r) {
        uint4 v = buf[(i + r * 37) & 1023];
        acc.x ^= v.x; acc.y += v.y;
        if (HAMMER > 1) buf[(i + r * 53) & 1023] = acc;
      }
    }
    if (acc.x == 12345) buf[0] = acc;
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(M, N);
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < ksteps; ++k) {
#pragma unroll
        for (int acc = 0; acc < NACC; ++acc) {
          uint64_t ad, bd;
          if (SW) {  // 4 K16 steps per 128-byte swizzle row: advance 32 B
            ad = sdesc_sw128(a0 + (k >> 2) * 16384 + (k & 3) * 32);
            bd = sdesc_sw128(b0 + (k >> 2) * (N * 128) + (k & 3) * 32);
          } else {
            ad = sdesc(a0 + (k & 1) * 16 * (SBO / 16) + (OFF ? (k & 7) * OFF : 0), 11680, SBO);
            bd = sdesc(b0 + (k & 7) * N * 32, N * 16, 128);
          }
          if (TS) umma_ts(tmem + acc * N, tmem + 256 + (k & 7) * 8, bd, idesc, (it | k) ? 1u : 0u);
          else umma_bf16(tmem + acc * N, ad, bd, idesc, (it | k) ? 1u : 0u);
        }
        if (CE && (k % CE) == CE - 1) umma_commit(&bar2);   // per-step completion tracking
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
    stop = 1;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, int NACC, bool SW, int SBO = 128, int HAMMER = 0, int OFF = 0, int M = 128, int CE = 0, int TS = 0>
void run() {
  const int iters = 500, ksteps = 8;
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  size_t smem = 32768 + 8 * 256 * 32 + 2048;
  cudaFuncSetAttribute(mma_loop<N, NACC, SW, SBO, HAMMER, OFF, M, CE, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_loop<N, NACC, SW, SBO, HAMMER, OFF, M, CE, TS><<<148, 512, smem>>>(iters, ksteps, d);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("N=%d acc=%d sw=%d: %s\n", N, NACC, (int)SW, cudaGetErrorString(err)); fflush(stdout); return; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<N, NACC, SW, SBO, HAMMER, OFF, M, CE, TS><<<148, 512, smem>>>(iters, ksteps, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mmas = (double)iters * ksteps * NACC;
  double flops = mmas * 2.0 * M * N * 16 * 148;
  printf("%s CE=%d M=%3d H=%d OFF=%3d SBO=%3d N=%3d acc=%d %s: %6.2f cycles/MMA (floor %3d), %7.1f TFLOP/s  %s\n", TS ? "TS" : "SS", CE, M, HAMMER, OFF, SBO, N, NACC,
         SW ? "SW128" : "none ", (double)h[0] / mmas, M * N / 256, flops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  cudaFree(d);
}

int main() {
  // N = 64, SS mode: 1..4 interleaved accumulators (the fused conv2 shape)
  run<64, 1, false, 128, 0, 0, 128, 0, 0>(); run<64, 2, false, 128, 0, 0, 128, 0, 0>();
  run<64, 3, false, 128, 0, 0, 128, 0, 0>(); run<64, 4, false, 128, 0, 0, 128, 0, 0>();
  run<64, 3, false, 432, 0, 16, 128, 0, 0>();
  return 0;
}
