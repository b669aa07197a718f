// gemm_tc.cu — fp32-accurate GEMM on the tcgen05 tensor cores, the contraction
// of the specialized-CNN training path (train.cu):
//   C[m][n] = sum_k A(m, k) B(k, n),  A(m, k) = A[m*sam + k*sak], B(k, n) = B[n*sbn + k*sbk]
// (any strides, so every op(A) op(B) of the backward pass is one call, no
// transposes in memory).  Precision: "3xTF32" — each fp32 operand x is split
// into x_hi = tf32_rna(x) and x_lo = x - x_hi, and the tensor core accumulates
// a_hi b_hi + a_hi b_lo + a_lo b_hi in fp32 (the a_lo b_lo term is below fp32
// rounding), which keeps the result at fp32 accuracy (R-25: training runs in fp32).
//
// CTA tile 128 x BN (BN in {32, 64, 128}), K in stages of 32 (16 for BN = 128): 256
// threads load a stage of A and B (all loads in flight before any store), split it
// and store it into the canonical no-swizzle K-major shared-memory layout (core
// matrix = 8 rows x 4 tf32; a warp fills one core matrix per store, bank-conflict
// free); one elected thread issues the K-steps x 3 tcgen05.mma.kind::tf32 into the
// TMEM accumulator, double-buffered against the next stage's loads (mbarrier per
// stage); the epilogue stages each warp's 32 x 16 block through shared memory so the
// global stores are row segments.  Split-K over blockIdx.z writes fp32 partials that
// a second kernel sums in a fixed order (deterministic, no atomics).
#include "common.cuh"
#include "internal.h"

namespace ns {

namespace {
constexpr int kGT = 256;           // threads per CTA (8 warps: loads / splits / stores)
constexpr int kBM = 128, kBK = 32;   // kBK: host-side chunk granularity (split-K ranges)

// Instruction descriptor: kind::tf32, A/B tf32, D fp32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32_f32(int M, int N) {
  return (1u << 4)                         // c_format = F32
         | (2u << 7)                       // a_format = TF32
         | (2u << 10)                      // b_format = TF32
         | ((uint32_t)(N >> 3) << 17)      // n_dim
         | ((uint32_t)(M >> 4) << 24);     // m_dim
}
NS_DEV void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
NS_DEV float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// K-major canonical tile of `rows` rows x 32 k: core matrix (8-row group g, 4-element K
// chunk c) at byte ((c * rows/8) + g) * 128; element (r, k) at + (r % 8) * 16 + (k % 4) * 4

template <int BN>
struct GemmSmem {
  static constexpr int BK = BN == 128 ? 16 : 32;   // K per stage (BN = 128: 2 CTAs / SM)
  static constexpr int kKSteps = BK / 8;           // tf32 MMA K = 8
  static constexpr int kA = kBM * BK * 4;
  static constexpr int kB = BN * BK * 4;
  static constexpr int kStage = 2 * kA + 2 * kB;   // hi + lo of A and B
  static constexpr int kBytes = 2 * kStage + 64;
};

template <int BN>
__global__ void __launch_bounds__(kGT)
gemm3xtf32_kernel(TcGemmArgs G) {
  using S = GemmSmem<BN>;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* done = reinterpret_cast<uint64_t*>(sm + 2 * S::kStage);   // [2] MMA commit per stage
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
  const int64_t k0 = (int64_t)blockIdx.z * G.kper, k1 = min((int64_t)G.K, k0 + G.kper);
  if (tid == 0) {
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_rt(tslot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = idesc_tf32_f32(kBM, BN);
  const int nchunks = (int)((k1 - k0 + S::BK - 1) / S::BK);
  for (int it = 0; it < nchunks; ++it) {
    const int s = it & 1;
    uint8_t* st = sm + s * S::kStage;
    float* ahi = reinterpret_cast<float*>(st);
    float* alo = reinterpret_cast<float*>(st + S::kA);
    float* bhi = reinterpret_cast<float*>(st + 2 * S::kA);
    float* blo = reinterpret_cast<float*>(st + 2 * S::kA + S::kB);
    const int64_t kb = k0 + (int64_t)it * S::BK;
    // All of this thread's global loads first (memory-level parallelism), then the tf32
    // split and the stores.  A warp fills one core matrix (8 rows x 4 k = 128 B) per
    // step: lane -> (row 8g + lane/4, k 4c + lane%4), core matrix cm = c * rows/8 + g
    // at byte cm * 128, so the shared-memory stores are 32 consecutive words (no bank
    // conflicts) and the global loads are 8 segments of 16 B (rows) or 4 of 32 B (k).
    constexpr int kPA = kBM * S::BK / kGT, kPB = BN * S::BK / kGT;
    const int lane = tid & 31, wq = tid >> 5;
    float va[kPA], vb[kPB];
#pragma unroll
    for (int i = 0; i < kPA; ++i) {
      const int cm = wq + i * (kGT / 32);
      const int r = 8 * (cm % (kBM / 8)) + (lane >> 2), k = 4 * (cm / (kBM / 8)) + (lane & 3);
      const int m = m0 + r;
      const int64_t kk = kb + k;
      va[i] = (m < G.M && kk < k1) ? __ldg(G.A + (int64_t)m * G.sam + kk * G.sak) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < kPB; ++i) {
      const int cm = wq + i * (kGT / 32);
      const int r = 8 * (cm % (BN / 8)) + (lane >> 2), k = 4 * (cm / (BN / 8)) + (lane & 3);
      const int n = n0 + r;
      const int64_t kk = kb + k;
      vb[i] = (n < G.N && kk < k1) ? __ldg(G.B + (int64_t)n * G.sbn + kk * G.sbk) : 0.0f;
    }
    if (it >= 2) mbar_wait(&done[s], (uint32_t)(((it >> 1) - 1) & 1));   // stage s free again
#pragma unroll
    for (int i = 0; i < kPA; ++i) {
      const int o = (wq + i * (kGT / 32)) * 32 + lane;   // float index = cm * 32 + lane
      const float hi = tf32_rna(va[i]);
      ahi[o] = hi;
      alo[o] = va[i] - hi;
    }
#pragma unroll
    for (int i = 0; i < kPB; ++i) {
      const int o = (wq + i * (kGT / 32)) * 32 + lane;
      const float hi = tf32_rna(vb[i]);
      bhi[o] = hi;
      blo[o] = vb[i] - hi;
    }
    fence_proxy_async_smem();   // generic-proxy stores -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = smem_u32(ahi), sal = smem_u32(alo), sb = smem_u32(bhi), sbl = smem_u32(blo);
      // K-major canonical: LBO = next 4-element K chunk = rows/8 core matrices, SBO = 128 B
      const uint32_t lboA = (kBM / 8) * 128, lboB = (BN / 8) * 128;
#pragma unroll
      for (int ks = 0; ks < S::kKSteps; ++ks) {
        const uint32_t oa = (uint32_t)(2 * ks) * lboA, ob = (uint32_t)(2 * ks) * lboB;
        const uint64_t dah = sdesc(sa + oa, lboA, 128), dal = sdesc(sal + oa, lboA, 128);
        const uint64_t dbh = sdesc(sb + ob, lboB, 128), dbl = sdesc(sbl + ob, lboB, 128);
        const uint32_t acc0 = (it > 0 || ks > 0) ? 1u : 0u;
        umma_tf32(tmem, dah, dbh, idesc, acc0);
        umma_tf32(tmem, dah, dbl, idesc, 1u);
        umma_tf32(tmem, dal, dbh, idesc, 1u);
      }
      umma_commit(&done[s]);
    }
  }
  // drain: the last commit covers every earlier MMA
  if (nchunks > 0) mbar_wait(&done[(nchunks - 1) & 1], (uint32_t)(((nchunks - 1) >> 1) & 1));
  tc_fence_after();
  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 (its lane quarter), warps
  // w and w + 4 split the accumulator columns
  const int quarter = warp & 3, half = warp >> 2;
  float* out = G.part ? G.part + (int64_t)blockIdx.z * G.M * G.N : G.C;
  const int64_t ldo = G.part ? G.N : G.ldc;
  constexpr int kColsPerHalf = BN / 2;
  // stores staged per warp through shared memory (the stage buffers are free now):
  // 32 rows x 16 columns written by row, read back two rows per instruction so a
  // warp's global stores are two contiguous 64-byte row segments
  __syncthreads();
  float* stage = reinterpret_cast<float*>(sm) + warp * (32 * 17);
  const int lane = tid & 31;
#pragma unroll 1
  for (int c = half * kColsPerHalf; c < (half + 1) * kColsPerHalf; c += 16) {
    uint32_t r[16];
    if (nchunks > 0) {
      tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + c, r);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = 0u;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) stage[lane * 17 + j] = __uint_as_float(r[j]);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int rr = 2 * i + (lane >> 4), cc = lane & 15;
      const int mm = m0 + quarter * 32 + rr, n = n0 + c + cc;
      if (mm < G.M && n < G.N) out[(int64_t)mm * ldo + n] = stage[rr * 17 + cc];
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc_rt(tmem, BN);
}

// C = sum of the split-K partials: one warp per output element, lanes take the
// splits z = lane, lane + 32, ... and a fixed shuffle tree combines them
// (deterministic: the same order every run).
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int ksplit, int M, int N, float* __restrict__ C,
                                     int64_t ldc) {
  const int64_t total = (int64_t)M * N;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = w0; e < total; e += nw) {
    float s = 0.0f;
    for (int z = lane; z < ksplit; z += 32) s += part[(int64_t)z * total + e];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) C[(e / N) * ldc + e % N] = s;
  }
}

template <int BN>
noscope_status launch_bn(TcGemmArgs g, cudaStream_t st) {
  using S = GemmSmem<BN>;
  static DeviceOnce attr;
  if (attr.first())
    NS_CUDA_TRY(cudaFuncSetAttribute(gemm3xtf32_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes));
  const dim3 grid((unsigned)((g.M + kBM - 1) / kBM), (unsigned)((g.N + BN - 1) / BN), (unsigned)g.ksplit);
  gemm3xtf32_kernel<BN><<<grid, kGT, S::kBytes, st>>>(g);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}
}  // namespace

size_t tc_gemm_part_floats(int M, int N, int64_t K) {
  const int64_t tiles = (int64_t)((M + kBM - 1) / kBM) * ((N + 127) / 128);
  const int64_t chunks = (K + kBK - 1) / kBK;
  // split K when the output has few tiles and the reduction is long (the weight gradients)
  int ks = 1;
  while (tiles * ks < 2 * kNumSMs && chunks / (ks * 2) >= 4 && ks < 256) ks *= 2;
  return ks > 1 ? (size_t)ks * M * N : 0;
}

static noscope_status run_gemm(TcGemmArgs g, float* part, cudaStream_t st) {
  const int M = g.M, N = g.N;
  const int64_t K = g.K;
  if (M <= 0 || N <= 0) return NOSCOPE_OK;
  const int BN = N <= 32 ? 32 : (N <= 64 ? 64 : 128);
  const int64_t tiles = (int64_t)((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int64_t chunks = (K + kBK - 1) / kBK;
  int ks = 1;
  while (tiles * ks < 2 * kNumSMs && chunks / (ks * 2) >= 4 && ks < 256) ks *= 2;
  if (ks > 1 && !part) ks = 1;
  g.ksplit = ks;
  g.kper = ((chunks + ks - 1) / ks) * kBK;
  g.part = ks > 1 ? part : nullptr;
  noscope_status s = BN == 32 ? launch_bn<32>(g, st) : (BN == 64 ? launch_bn<64>(g, st) : launch_bn<128>(g, st));
  if (s != NOSCOPE_OK || ks == 1) return s;
  const int64_t total = (int64_t)M * N;
  splitk_reduce_kernel<<<(int)std::min<int64_t>((total * 32 + 255) / 256, 16 * kNumSMs), 256, 0, st>>>(
      part, ks, M, N, g.C, g.ldc);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

noscope_status tc_gemm(const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn, int64_t sbk, float* C,
                       int64_t ldc, int M, int N, int64_t K, float* part, cudaStream_t st) {
  TcGemmArgs g{};
  g.A = A; g.sam = sam; g.sak = sak;
  g.B = B; g.sbn = sbn; g.sbk = sbk;
  g.C = C; g.ldc = ldc;
  g.M = M; g.N = N; g.K = K;
  return run_gemm(g, part, st);
}

}  // namespace ns
