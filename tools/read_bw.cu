// Streaming-read bandwidth ceiling on this B200: each thread reads uint4s in a
// grid-stride loop (plain ld.global and ld.global.cs variants) and folds them into
// one word so the loads cannot be dropped.  Reports GB/s of bytes read.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool CS>
__global__ void rd(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = CS ? __ldcs(p + i) : p[i];
    acc ^= v.x + v.y + v.z + v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}

int main() {
  const size_t bytes = 16ull << 30, n = bytes / 16;
  uint4* p;
  unsigned* o;
  cudaMalloc(&p, bytes);
  cudaMalloc(&o, 4);
  cudaMemset(p, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int cs = 0; cs < 2; ++cs)
    for (int bpsm : {2, 4, 8, 16}) {
      const int grid = 148 * bpsm;
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        if (cs) rd<true><<<grid, 512>>>(p, n, o); else rd<false><<<grid, 512>>>(p, n, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("cs=%d blocks/SM=%2d: %.1f GB/s\n", cs, bpsm, bytes / best / 1e6);
    }
  return 0;
}
