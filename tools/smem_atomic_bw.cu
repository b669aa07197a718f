// Shared-memory atomic and load throughput on this B200 (the ceilings of the
// sweep histogram kernel, sweep_hist_kernel): one CTA per SM x 512 threads,
// each thread issues K operations on addresses drawn from a hash of (thread, i)
// over a region of W u32 words (W = 41,616 is the sweep's 100 x 100 candidate
// histogram; W = 32 / same-address / distinct-bank patterns for reference).
// Reports operations per clock per SM (SM clock read with clock64 in-kernel)
// and per second for the whole GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smem_atomic_bw tools/smem_atomic_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// mode 0: random words in [0, W)   mode 1: word = lane (conflict-free)
// mode 2: every lane the same word  mode 3: random u32 LOADS (no atomics)
// mode 4: random 8-byte loads over W/2 doubles (the binary-search access)
template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(int W, int K, unsigned long long* cycles, unsigned* sink) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) h[i] = i;
  __syncthreads();
  const uint32_t seed = mix(blockIdx.x * 4096 + threadIdx.x);
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int i = 0; i < K; ++i) {
    const uint32_t r = mix(seed + i * 0x9e3779b9u);
    if (MODE == 0) atomicAdd(&h[r % W], 1u);
    if (MODE == 1) atomicAdd(&h[threadIdx.x & 31], 1u);
    if (MODE == 2) atomicAdd(&h[0], 1u);
    if (MODE == 3) acc += h[r % W];
    if (MODE == 4) acc += (uint32_t)reinterpret_cast<const double*>(h)[r % (W / 2)];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345u) sink[0] = acc;
}

template <int MODE>
void run(const char* name, int W, int K) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  unsigned* sink;
  cudaMalloc(&cyc, sms * 8);
  cudaMalloc(&sink, 4);
  const size_t smem = (size_t)W * 4;
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<MODE><<<sms, 512, smem>>>(W, K / 10, cyc, sink);   // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE><<<sms, 512, smem>>>(W, K, cyc, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += (double)h[i] / sms;
  const double ops = 512.0 * K;   // per SM
  printf("%-34s W=%6d  %.3f ops/clk/SM  %.2f Gops/s GPU  (%.3f ms, %.0f cycles)\n", name, W, ops / mean,
         ops * sms / (ms * 1e-3) / 1e9, ms, mean);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  const int K = 20000;
  run<0>("atomicAdd u32, random word", 41616, K);
  run<0>("atomicAdd u32, random word", 4096, K);
  run<1>("atomicAdd u32, word = lane", 32, K);
  run<2>("atomicAdd u32, same word", 32, K);
  run<3>("ld.shared u32, random word", 41616, K);
  run<4>("ld.shared f64, random of 128", 256, K);
  run<4>("ld.shared f64, random of 20808", 41616, K);
  return 0;
}
