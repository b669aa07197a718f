// Ceiling of dd_kernel's loading structure: persistent CTAs stream a contiguous range of
// 640x480x3 frames as per-output-row bands (cp.async.bulk, one mbarrier per stage) through
// an S-stage shared-memory ring; consumer warps optionally read every byte (LDS.128) and
// release the stage through an "empty" mbarrier.  Reports GB/s of source bytes streamed
// for a sweep of (CTAs per SM, stages, band split, consumer reads).  No compute: the gap
// between this and dd_kernel is the cost of its V/H work and synchronisation.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1703_02529_b200/csrc/common.cuh"
using namespace ns;

struct Args {
  const uint8_t* frames;
  int64_t n_frames, pitch;
  int band_bytes, bands_per_frame, split, stages, read;
  unsigned* sink;
};

__global__ void __launch_bounds__(256) ring(Args A) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 16;
  uint8_t* stage = smem + 256;
  const int64_t f0 = A.n_frames * blockIdx.x / gridDim.x, f1 = A.n_frames * (blockIdx.x + 1) / gridDim.x;
  const int64_t total = (f1 - f0) * A.bands_per_frame;
  const int nw = blockDim.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < A.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nw - 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int sb = A.band_bytes;
  if (threadIdx.x / 32 == 0) {  // producer warp
    if (threadIdx.x != 0) return;
    const uint64_t pol = policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    for (int64_t q = 0; q < total; ++q) {
      if (q >= A.stages) mbar_wait(&empty[s], ph ^ 1u);
      const int64_t f = f0 + q / A.bands_per_frame;
      const int bi = (int)(q % A.bands_per_frame);
      const uint8_t* src = A.frames + f * A.pitch + (int64_t)bi * sb;
      mbar_arrive_expect_tx(&full[s], (uint32_t)sb);
      const int part = sb / A.split;
      for (int p = 0; p < A.split; ++p)
        bulk_g2s_evict_first(stage + (size_t)s * sb + p * part, src + p * part, (uint32_t)part, &full[s], pol);
      if (++s == A.stages) { s = 0; ph ^= 1u; }
    }
    return;
  }
  const int ct = threadIdx.x - 32, nct = blockDim.x - 32;
  int s = 0;
  uint32_t ph = 0, acc = 0;
  for (int64_t q = 0; q < total; ++q) {
    mbar_wait(&full[s], ph);
    if (A.read) {
      const uint4* p = reinterpret_cast<const uint4*>(stage + (size_t)s * sb);
      for (int u = ct; u < sb / 16; u += nct) {
        const uint4 v = p[u];
        acc ^= v.x + v.y + v.z + v.w;
      }
    }
    __syncwarp();
    if ((ct & 31) == 0) mbar_arrive(&empty[s]);
    if (++s == A.stages) { s = 0; ph ^= 1u; }
  }
  if (acc == 0x12345678u) *A.sink = acc;
}

int main() {
  const int W = 640, H = 480;
  const int64_t pitch = (int64_t)W * H * 3;
  const int64_t n = 108000;
  uint8_t* fr;
  unsigned* sink;
  if (cudaMalloc(&fr, n * pitch) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&sink, 4);
  cudaMemset(fr, 1, n * pitch);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg { int bpf, cps, stages, split, read; };
  // band = pitch / bpf bytes (bpf = 48 -> 19,200 B like dd_kernel's 10-row bands)
  const Cfg cfgs[] = {
      {48, 2, 5, 1, 1}, {48, 2, 5, 1, 0}, {48, 2, 4, 1, 1}, {48, 2, 5, 4, 1}, {48, 3, 3, 1, 1},
      {48, 3, 3, 1, 0}, {48, 4, 2, 1, 1}, {96, 2, 10, 1, 1}, {96, 3, 7, 1, 1}, {96, 4, 5, 1, 1},
      {96, 6, 3, 1, 1}, {192, 4, 10, 1, 1}, {192, 6, 7, 1, 1}, {192, 8, 5, 1, 1}, {24, 2, 2, 1, 1},
      {24, 1, 5, 1, 1}, {48, 1, 10, 1, 1}, {48, 1, 8, 1, 1}, {48, 1, 6, 1, 1}, {48, 1, 9, 1, 1},
      {48, 1, 11, 1, 1}};
  for (const Cfg& c : cfgs) {
    Args A{fr, n, pitch, (int)(pitch / c.bpf), c.bpf, c.split, c.stages, c.read, sink};
    const size_t smem = 256 + (size_t)c.stages * A.band_bytes;
    if (smem > (227 * 1024) / c.cps - 1024) { printf("bpf %d cps %d stages %d: smem %zu too big\n", c.bpf, c.cps, c.stages, smem); continue; }
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a);
      ring<<<148 * c.cps, 256, smem>>>(A);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("band %6d B  ctas/SM %d  stages %2d  split %d  read %d  smem %6zu : %7.3f ms  %7.1f GB/s %s\n",
           A.band_bytes, c.cps, c.stages, c.split, c.read, smem, best, n * pitch / best / 1e6,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
