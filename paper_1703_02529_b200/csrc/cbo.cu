// cbo.cu — device helper of the full CBO search:
// the per-frame label a_i the cascade would emit for frame i if it is NOT fired
// (the oracle's build_records): skipped -> label of its period's checked
// frame; checked and suppressed -> 0 (reference-image DD) or label(t - k)
// (earlier-frame DD; 0 before the first anchor).  The search itself
// (noscope_cbo_search) sequences the existing DD / CNN / sweep launches.
#include "common.cuh"
#include "internal.h"

namespace ns {

__global__ void records_a_kernel(const double* __restrict__ score, const uint8_t* __restrict__ y,
                                 int64_t n, int mode, int k, int t_skip, uint8_t* __restrict__ a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (score[i] == __longlong_as_double(0xFFF0000000000000ll)) {   // -inf: skipped
      a[i] = y[i - i % t_skip];
    } else {
      a[i] = (mode == 0 || i < k) ? 0 : y[i - k];
    }
  }
}

noscope_status launch_records_a(const double* score, const uint8_t* y, int64_t n, int mode, int k,
                                int t_skip, uint8_t* a, cudaStream_t st) {
  if (n == 0) return NOSCOPE_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 4 * kNumSMs);
  records_a_kernel<<<grid, 256, 0, st>>>(score, y, n, mode, k, t_skip, a);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

}  // namespace ns

namespace ns {
// ---------------------------------------------------------------- evaluation
// Windowed accuracy (30-frame windows, correct iff >= 28 agree) and
// frame confusion counts in one pass; counters[0..5] = windows, correct windows,
// tp, tn, fp, fn (u64, zeroed by the caller).
__global__ void eval_labels_kernel(const uint8_t* __restrict__ pred, const uint8_t* __restrict__ ref,
                                   int64_t n, int window, int agree_min,
                                   unsigned long long* __restrict__ counters) {
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  const int64_t nw = n / window;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
    int agree = 0;
    for (int j = 0; j < window; ++j) agree += ((pred[w * window + j] != 0) == (ref[w * window + j] != 0));
    c[0] += 1;
    c[1] += agree >= agree_min;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool p = pred[i] != 0, r = ref[i] != 0;
    c[2] += p && r;
    c[3] += !p && !r;
    c[4] += p && !r;
    c[5] += !p && r;
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const unsigned long long v = warp_sum(c[q]);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&counters[q], v);
  }
}

// The paper's 30-frame windows, one pass: a thread owns blocks of 16 windows = 480 bytes =
// 30 aligned 16-byte vectors of each track (grid-stride over blocks); per vector, the
// agreement / confusion bits of its 16 frames are formed with byte-SIMD compares and
// each frame's agreement is added to its window (compile-time window of every byte, the
// vector loop is unrolled); frames after the last whole block take the generic loop.
NS_DEV uint32_t nz_bytes(uint32_t x) {   // 0x01 in every byte of x that is nonzero
  return (__vcmpne4(x, 0u) & 0x01010101u);
}
__global__ void eval_labels30_kernel(const uint8_t* __restrict__ pred, const uint8_t* __restrict__ ref,
                                     int64_t n, int agree_min, unsigned long long* __restrict__ counters) {
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  const int64_t nb = n / 480;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
    const uint4* P = reinterpret_cast<const uint4*>(pred + b * 480);
    const uint4* R = reinterpret_cast<const uint4*>(ref + b * 480);
    uint32_t agree[16];
#pragma unroll
    for (int w = 0; w < 16; ++w) agree[w] = 0;
    uint32_t tp = 0, tn = 0, fp = 0, fnn = 0;
#pragma unroll
    for (int q = 0; q < 30; ++q) {
      const uint4 pv = __ldcs(P + q), rv = __ldcs(R + q);
      const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w}, rw[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t pb = nz_bytes(pw[j]), rb = nz_bytes(rw[j]);
        const uint32_t both = pb & rb, none = (pb | rb) ^ 0x01010101u;
        tp += __popc(both);
        tn += __popc(none);
        fp += __popc(pb & ~rb);
        fnn += __popc(rb & ~pb);
        const uint32_t ag = both | none;   // 0x01 per agreeing frame
#pragma unroll
        for (int e = 0; e < 4; ++e) agree[(16 * q + 4 * j + e) / 30] += (ag >> (8 * e)) & 1u;
      }
    }
    c[0] += 16;
#pragma unroll
    for (int w = 0; w < 16; ++w) c[1] += agree[w] >= (uint32_t)agree_min;
    c[2] += tp;
    c[3] += tn;
    c[4] += fp;
    c[5] += fnn;
  }
  // the tail after the last whole 480-frame block: generic per-frame / per-window loops
  const int64_t t0 = nb * 480, nw = n / 30;
  for (int64_t w = t0 / 30 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
    int agree = 0;
    for (int j = 0; j < 30; ++j) agree += ((pred[w * 30 + j] != 0) == (ref[w * 30 + j] != 0));
    c[0] += 1;
    c[1] += agree >= agree_min;
  }
  for (int64_t i = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool p = pred[i] != 0, r = ref[i] != 0;
    c[2] += p && r;
    c[3] += !p && !r;
    c[4] += p && !r;
    c[5] += !p && r;
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const unsigned long long v = warp_sum(c[q]);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&counters[q], v);
  }
}

noscope_status launch_eval_labels(const uint8_t* pred, const uint8_t* ref, int64_t n, int window,
                                  int agree_min, unsigned long long* counters, int64_t* out_host,
                                  cudaStream_t st) {
  NS_CUDA_TRY(cudaMemsetAsync(counters, 0, 6 * 8, st));
  if (n > 0) {
    const bool v30 = window == 30 && ((reinterpret_cast<uintptr_t>(pred) | reinterpret_cast<uintptr_t>(ref)) & 15) == 0;
    if (v30) {
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n / 480 + 255) / 256, 8 * kNumSMs));
      eval_labels30_kernel<<<grid, 256, 0, st>>>(pred, ref, n, agree_min, counters);
    } else {
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4 * kNumSMs));
      eval_labels_kernel<<<grid, 256, 0, st>>>(pred, ref, n, window, agree_min, counters);
    }
    NS_LAUNCH_CHECK();
    count_launch();
  }
  NS_CUDA_TRY(cudaMemcpyAsync(out_host, counters, 6 * 8, cudaMemcpyDeviceToHost, st));
  NS_CUDA_TRY(cudaStreamSynchronize(st));
  return NOSCOPE_OK;
}
}  // namespace ns
