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
