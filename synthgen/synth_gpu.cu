// synth_gpu.cu — GPU renderer of the synthetic fixed-angle video and the
// ground-truth stand-in labeller.  HARNESS code (input generation), not part
// of NoScope's method: it reproduces synthgen/__init__.py byte for byte
// (splitmix64 counter hash; tests/test_synthgen.py checks equality).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One CTA per (frame, row).  bg: uint8 [H][W][3] static background (rendered
// by bg_kernel); events int32 [E][10]; active int32 [T][3] for the unit.
__global__ void render_kernel(uint8_t* out, int64_t pitch, int W, int H, int64_t t_begin,
                              int64_t n, uint64_t seed, uint64_t stream, int sigma,
                              const uint8_t* bg, const int32_t* events, const int32_t* active) {
  const int64_t fr = blockIdx.x / H;
  const int y = blockIdx.x % H;
  if (fr >= n) return;
  const int64_t t = t_begin + fr;
  uint64_t k = sm64(seed);
  k = sm64(k ^ stream);
  k = sm64(k ^ ((1ull << 32) + (uint64_t)t));
  k = sm64(k ^ (uint64_t)y);
  int rect[3][5];  // xa, xb (clipped), color
  int nr = 0;
  for (int s = 0; s < 3; ++s) {
    const int e = active[t * 3 + s];
    if (e < 0) continue;
    const int32_t* ev = events + (int64_t)e * 10;
    const int dt = (int)(t - ev[0]);
    const int x = ev[2] + ev[4] * dt, yy = ev[3] + ev[5] * dt;
    if (y < yy || y >= yy + ev[7]) continue;
    rect[nr][0] = x;
    rect[nr][1] = x + ev[6];
    rect[nr][2] = ev[8];
    ++nr;
  }
  uint8_t* row = out + fr * pitch + (int64_t)y * W * 3;
  const uint8_t* brow = bg + (int64_t)y * W * 3;
  const int span = 2 * sigma + 1;
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    int base[3] = {brow[x * 3], brow[x * 3 + 1], brow[x * 3 + 2]};
    for (int r = 0; r < nr; ++r)
      if (x >= rect[r][0] && x < rect[r][1]) {
        base[0] = rect[r][2] & 0xFF;
        base[1] = (rect[r][2] >> 8) & 0xFF;
        base[2] = (rect[r][2] >> 16) & 0xFF;
      }
    if (sigma > 0) {
      const uint64_t h = sm64(k ^ (uint64_t)x);
      for (int c = 0; c < 3; ++c) base[c] += (int)(((h >> (16 * c)) & 0xFFFF) % span) - sigma;
    }
    for (int c = 0; c < 3; ++c) {
      int v = base[c] < 0 ? 0 : (base[c] > 255 ? 255 : base[c]);
      row[x * 3 + c] = (uint8_t)v;
    }
  }
}

__global__ void bg_kernel(uint8_t* bg, int W, int H, uint64_t seed, uint64_t stream) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)W * H) return;
  const int y = (int)(p / W), x = (int)(p % W);
  uint64_t k = sm64(seed);
  k = sm64(k ^ stream);
  k = sm64(k ^ 1ull);
  k = sm64(k ^ (uint64_t)y);
  const uint64_t h = sm64(k ^ (uint64_t)x);
  for (int c = 0; c < 3; ++c) bg[p * 3 + c] = (uint8_t)(40 + ((h >> (16 * c)) & 0xFFFF) % 101);
}

__global__ void truth_kernel(const uint8_t* truth, const int32_t* idx, const int64_t* n_dev,
                             int64_t n_max, int64_t base, uint8_t* answers) {
  const int64_t n = n_dev ? (*n_dev < n_max ? *n_dev : n_max) : n_max;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    answers[i] = truth[base + idx[i]];
}

}  // namespace

extern "C" {

int synth_render_bg(uint8_t* bg, int W, int H, uint64_t seed, uint64_t stream, cudaStream_t s) {
  const int64_t n = (int64_t)W * H;
  bg_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(bg, W, H, seed, stream);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
}

int synth_render(uint8_t* out, int64_t pitch, int W, int H, int64_t t_begin, int64_t n,
                 uint64_t seed, uint64_t stream, int sigma, const uint8_t* bg,
                 const int32_t* events, const int32_t* active, cudaStream_t s) {
  if (n <= 0) return 0;
  render_kernel<<<(unsigned)(n * H), 256, 0, s>>>(out, pitch, W, H, t_begin, n, seed, stream, sigma,
                                                   bg, events, active);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
}

// noscope_labeller_fn-compatible stand-in for the reference network: looks up
// ground-truth labels (user = device uint8 truth track indexed by absolute frame).
int synth_truth_labeller(void* user, const int32_t* idx, const int64_t* n_dev, int64_t n_max,
                         int64_t base, uint8_t* answers, cudaStream_t s) {
  if (n_max <= 0) return 0;
  int grid = (int)((n_max + 255) / 256);
  if (grid > 1184) grid = 1184;
  truth_kernel<<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(user), idx, n_dev, n_max, base,
                                    answers);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 1;
}

}  // extern "C"
