// Unit test: tcgen05.mma kind::f16 with the A operand in TENSOR MEMORY
// ("TS" form).  Hypothesis under test: A (M=128 x K=16, bf16) occupies lanes
// 0..127 = rows and 8 consecutive 32-bit columns, column c holding
// (A[m][2c] low half, A[m][2c+1] high half).  Compares D = A * B^T against the
// SS form (A from smem) and a host reference.  Also times TS vs SS at N = 32/64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_ts_test tools/umma_ts_test.cu
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../paper_1703_02529_b200/csrc/common.cuh"

using namespace ns;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

template <int N>
__global__ void ts_kernel(const uint16_t* Ag /*[128][16]*/, const uint16_t* Bg /*[N][16]*/,
                          float* Dts, float* Dss, int reps, long long* cyc) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];
  __shared__ __align__(1024) uint8_t sB[N * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // canonical K-major no-swizzle smem copies: [2 chunks][rows][8]
  for (int e = tid; e < 128 * 16; e += blockDim.x) {
    int m = e / 16, k = e % 16;
    reinterpret_cast<uint16_t*>(sA)[(k / 8) * 128 * 8 + m * 8 + (k % 8)] = Ag[e];
  }
  for (int e = tid; e < N * 16; e += blockDim.x) {
    int n = e / 16, k = e % 16;
    reinterpret_cast<uint16_t*>(sB)[(k / 8) * N * 8 + n * 8 + (k % 8)] = Bg[e];
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<256>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  // A into TMEM columns [192, 200): row m = lane (warp's lane group)
  {
    const int m = (warp & 3) * 32 + lane;
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) v[c] = (uint32_t)Ag[m * 16 + 2 * c] | ((uint32_t)Ag[m * 16 + 2 * c + 1] << 16);
    tmem_st8(tm + ((uint32_t)((warp & 3) * 32) << 16) + 192, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t bd = sdesc(smem_u32(sB), N * 16, 128);
    const uint64_t ad = sdesc(smem_u32(sA), 2048 / 16 * 16 == 2048 ? 128 * 16 : 0, 128);
    umma_ts(tm + 0, tm + 192, bd, idesc, 0);
    umma_bf16(tm + 64, ad, bd, idesc, 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    // timing: TS vs SS, 2 accumulators interleaved
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      umma_ts(tm + 0, tm + 192, bd, idesc, 1);
      umma_ts(tm + 64, tm + 192, bd, idesc, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 1);
    long long t1 = clock64();
    for (int r = 0; r < reps; ++r) {
      umma_bf16(tm + 0, ad, bd, idesc, 1);
      umma_bf16(tm + 64, ad, bd, idesc, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (reps == 0) {
    const int m = (warp & 3) * 32 + lane;
    uint32_t r[16];
    for (int cb = 0; cb < N / 16; ++cb) {
      tmem_ld16(tm + ((uint32_t)((warp & 3) * 32) << 16) + 0 + cb * 16, r);
      tmem_ld_wait();
      for (int j = 0; j < 16; ++j) Dts[m * N + cb * 16 + j] = __uint_as_float(r[j]);
      tmem_ld16(tm + ((uint32_t)((warp & 3) * 32) << 16) + 64 + cb * 16, r);
      tmem_ld_wait();
      for (int j = 0; j < 16; ++j) Dss[m * N + cb * 16 + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tm);
}

static uint16_t f2b(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float b2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

template <int N>
void test() {
  uint16_t hA[128 * 16], hB[N * 16];
  for (int i = 0; i < 128 * 16; ++i) hA[i] = f2b((float)((i * 37) % 17 - 8) / 8.0f);
  for (int i = 0; i < N * 16; ++i) hB[i] = f2b((float)((i * 53) % 13 - 6) / 4.0f);
  uint16_t *dA, *dB;
  float *dT, *dS;
  long long* dc;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dT, 128 * N * 4); cudaMalloc(&dS, 128 * N * 4); cudaMalloc(&dc, 16);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  ts_kernel<N><<<1, 128>>>(dA, dB, dT, dS, 0, dc);
  cudaError_t e = cudaDeviceSynchronize();
  float hT[128 * N], hS[128 * N];
  cudaMemcpy(hT, dT, sizeof(hT), cudaMemcpyDeviceToHost);
  cudaMemcpy(hS, dS, sizeof(hS), cudaMemcpyDeviceToHost);
  double mt = 0, ms = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < 16; ++k) ref += (double)b2f(hA[m * 16 + k]) * b2f(hB[n * 16 + k]);
      mt = fmax(mt, fabs(ref - hT[m * N + n]));
      ms = fmax(ms, fabs(ref - hS[m * N + n]));
    }
  ts_kernel<N><<<148, 128>>>(dA, dB, dT, dS, 4000, dc);
  cudaDeviceSynchronize();
  long long hc[2];
  cudaMemcpy(hc, dc, 16, cudaMemcpyDeviceToHost);
  printf("N=%d: %s  max|TS-ref|=%.3g  max|SS-ref|=%.3g   TS %.1f cyc/MMA  SS %.1f cyc/MMA\n", N,
         cudaGetErrorString(e), mt, ms, hc[0] / 8000.0, hc[1] / 8000.0);
  fflush(stdout);
}

int main() {
  test<32>();
  test<64>();
  test<128>();
  return 0;
}
