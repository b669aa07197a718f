// fit.cu — the difference detector's fitting steps on the
// GPU: the reference image ("computes the reference image by averaging
// frames where the reference model returns no labels"), per-frame block-MSE
// features, and the blocked-LR weights ("trains a logistic regression
// (LR) classifier to weigh each block").  Readings R-21 / R-22
// (DESIGN.md): half-up rounding of the mean on the 50x50 small frames; LR by
// full-batch gradient descent on z-scored features.
//
// All reductions run in a fixed order (per-CTA partials over fixed row ranges,
// summed in CTA order by the last CTA to arrive), so results are bitwise
// reproducible run to run.
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace ns {

namespace {
constexpr int kFitThreads = 256;

// ------------------------------------------------------------ reference image
// Per-position sums over the negative frames.  Thread = one 16-byte vector of
// the small frame; a CTA takes a contiguous frame range, accumulates u32 sums in
// registers (<= 2^32 / 255 frames per CTA) and adds them to the u64 totals.
__global__ void __launch_bounds__(512)
ref_sum_kernel(const uint8_t* __restrict__ small, int64_t pitch, int nvec, const uint8_t* __restrict__ labels,
               int64_t n, unsigned long long* __restrict__ sums, unsigned long long* __restrict__ count) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t f0 = blockIdx.x * per, f1 = min(n, f0 + per);
  unsigned cnt = 0;
  for (int v0 = 0; v0 < nvec; v0 += blockDim.x) {
    const int v = v0 + threadIdx.x;
    uint32_t acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0;
    // 8 frames per step: their labels and (negative frames') vectors are loaded
    // before any is used, so each thread keeps 8 independent loads in flight
    for (int64_t fb = f0; fb < f1; fb += 8) {
      uint4 q[8];
      bool use[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t f = fb + u;
        use[u] = f < f1 && __ldg(labels + f) == 0;
        q[u] = (use[u] && v < nvec) ? __ldg(reinterpret_cast<const uint4*>(small + f * pitch) + v)
                                    : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (v0 == 0 && threadIdx.x == 0 && use[u]) ++cnt;
        const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] += (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
      }
    }
    if (v < nvec)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (acc[j]) atomicAdd(&sums[v * 16 + j], (unsigned long long)acc[j]);
  }
  if (threadIdx.x == 0 && cnt) atomicAdd(count, (unsigned long long)cnt);
}

// ref[p] = floor((2 S + m) / (2 m)) (round half up), m = #negatives
__global__ void ref_finish_kernel(const unsigned long long* __restrict__ sums,
                                  const unsigned long long* __restrict__ count, int bytes,
                                  uint8_t* __restrict__ ref) {
  const unsigned long long m = *count;
  if (m == 0) return;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < bytes; p += gridDim.x * blockDim.x)
    ref[p] = (uint8_t)((2 * sums[p] + m) / (2 * m));
}

// ------------------------------------------------------------ block features
// One CTA per frame (grid-stride).  A thread sums the integer SSD of one
// (image row, block column) segment — consecutive pixels of one LR block — and
// adds it with one 32-bit shared atomic (a block's SSD < 2^32 for 8-bit frames
// up to 2^32 / (3 * 255^2) pixels); MSE = SSD / (block pixels * 3) in fp64.
__global__ void __launch_bounds__(kFitThreads)
block_feat_kernel(const uint8_t* __restrict__ small, int64_t pitch, int out_w, int out_h, int grid,
                  int mode, const uint8_t* __restrict__ ref, int k, int64_t n, double* __restrict__ feats) {
  __shared__ unsigned ssd[kMaxGrid * kMaxGrid];
  const int sy = out_h / grid, sx = out_w / grid, nb = grid * grid;
  const int nseg = out_h * grid;
  for (int64_t f = blockIdx.x; f < n; f += gridDim.x) {
    double* row = feats + f * nb;
    if (mode == 1 && f < k) {
      for (int b = threadIdx.x; b < nb; b += blockDim.x) row[b] = __longlong_as_double(0x7FF8000000000000ll);
      continue;
    }
    const uint8_t* a = small + f * pitch;
    const uint8_t* r = mode == 0 ? ref : small + (f - k) * pitch;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) ssd[b] = 0;
    __syncthreads();
    for (int sgi = threadIdx.x; sgi < nseg; sgi += blockDim.x) {
      const int y = sgi / grid, bx = sgi - y * grid;
      const int x0 = bx * sx, x1 = (bx == grid - 1) ? out_w : x0 + sx;
      const uint8_t* pa = a + (y * out_w + x0) * 3;
      const uint8_t* pr = r + (y * out_w + x0) * 3;
      unsigned s = 0;
      for (int e = 0; e < (x1 - x0) * 3; ++e) {
        const int d = (int)pa[e] - (int)pr[e];
        s += (unsigned)(d * d);
      }
      atomicAdd(&ssd[min(y / sy, grid - 1) * grid + bx], s);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int by = b / grid, bx = b - by * grid;
      const int h = (by == grid - 1) ? out_h - by * sy : sy;
      const int w = (bx == grid - 1) ? out_w - bx * sx : sx;
      row[b] = (double)ssd[b] / (double)(h * w * 3);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ LR fit
struct LrWs {
  double* X;          // [d][n] z-scored features (column-major: coalesced rows)
  double* mu;         // [d]
  double* sd;         // [d]
  double* part;       // [nblk][d + 1] per-CTA partials
  double* wb;         // [d + 1] parameters (w..., b)
  unsigned* counter;  // last-CTA arrival counter
  unsigned* bad;      // non-finite feature / target flag
  double* cls;        // [2] sum of targets, for the one-class check
};

// per-CTA partial column sums over a fixed row range: pass 0 sums F, pass 1 sums
// (F - mu)^2.  The last CTA combines the partials in CTA order.
__global__ void __launch_bounds__(kFitThreads)
lr_stats_kernel(const double* __restrict__ F, const uint8_t* __restrict__ t, int64_t n, int d, int pass,
                LrWs W) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  for (int k = threadIdx.x; k <= d; k += blockDim.x) {
    double s = 0.0;
    if (k < d) {
      const double m = pass ? W.mu[k] : 0.0;
      for (int64_t i = r0; i < r1; ++i) {
        const double v = F[i * d + k];
        if (!isfinite(v)) atomicOr(W.bad, 1u);
        s += pass ? (v - m) * (v - m) : v;
      }
    } else if (pass == 0) {
      for (int64_t i = r0; i < r1; ++i) s += (double)(t[i] != 0);
    }
    W.part[(size_t)blockIdx.x * (d + 1) + k] = s;
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(W.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = threadIdx.x; k <= d; k += blockDim.x) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(&W.part[(size_t)b * (d + 1) + k]);
    if (k < d) {
      if (pass == 0) W.mu[k] = s / (double)n;
      else {
        const double sd = sqrt(s / (double)n);
        W.sd[k] = sd > 0.0 ? sd : 1.0;
      }
    } else if (pass == 0) {
      W.cls[0] = s;
    }
  }
  if (threadIdx.x == 0) *W.counter = 0u;
}

__global__ void lr_standardize_kernel(const double* __restrict__ F, int64_t n, int d, LrWs W) {
  const int64_t total = n * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int k = (int)(e - i * d);
    W.X[(size_t)k * n + i] = (F[e] - W.mu[k]) / W.sd[k];
  }
}

// One gradient-descent iteration: r_i = sigmoid(X_i w + b) - t_i over the CTA's
// rows, partial X^T r and sum r, then the last CTA sums the partials in CTA order
// and updates (w, b) in place.
__global__ void __launch_bounds__(kFitThreads)
lr_step_kernel(const uint8_t* __restrict__ t, int64_t n, int d, int64_t per, double lr, double l2,
               LrWs W) {
  extern __shared__ double sh[];
  double* w = sh;               // [d + 1]
  double* r = sh + (d + 1);     // [per]
  const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  for (int k = threadIdx.x; k <= d; k += blockDim.x) w[k] = W.wb[k];
  __syncthreads();
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double z = w[d];
    for (int k = 0; k < d; ++k) z += W.X[(size_t)k * n + i] * w[k];
    r[i - r0] = 1.0 / (1.0 + exp(-z)) - (double)(t[i] != 0);
  }
  __syncthreads();
  // partial X^T r over this CTA's rows: P = blockDim / (d + 1) threads per feature
  // take interleaved rows (4 independent accumulators each); the P sums are then
  // combined in p order — a fixed order, so the result is reproducible.
  double* red = r + per;   // [P][d + 1]
  const int P = max(1, (int)blockDim.x / (d + 1));
  for (int e = threadIdx.x; e < P * (d + 1); e += blockDim.x) {
    const int k = e % (d + 1), p = e / (d + 1);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double* xk = k < d ? W.X + (size_t)k * n : nullptr;
    int64_t i = r0 + p;
    for (; i + 3 * P < r1; i += 4 * P) {
      const double g0 = r[i - r0], g1 = r[i + P - r0], g2 = r[i + 2 * P - r0], g3 = r[i + 3 * P - r0];
      a0 += xk ? xk[i] * g0 : g0;
      a1 += xk ? xk[i + P] * g1 : g1;
      a2 += xk ? xk[i + 2 * P] * g2 : g2;
      a3 += xk ? xk[i + 3 * P] * g3 : g3;
    }
    for (; i < r1; i += P) a0 += xk ? xk[i] * r[i - r0] : r[i - r0];
    red[p * (d + 1) + k] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  for (int k = threadIdx.x; k <= d; k += blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < P; ++p) s += red[p * (d + 1) + k];
    W.part[(size_t)blockIdx.x * (d + 1) + k] = s;
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(W.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = threadIdx.x; k <= d; k += blockDim.x) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(&W.part[(size_t)b * (d + 1) + k]);
    const double g = s / (double)n + (k < d ? l2 * w[k] : 0.0);
    W.wb[k] = w[k] - lr * g;
  }
  if (threadIdx.x == 0) *W.counter = 0u;
}

// raw-feature parameters: w_raw = w / sd, b_raw = b - sum_k w_k mu_k / sd_k (k order)
__global__ void lr_unscale_kernel(int d, LrWs W, double* out) {
  if (threadIdx.x != 0) return;
  double b = W.wb[d];
  for (int k = 0; k < d; ++k) {
    out[k] = W.wb[k] / W.sd[k];
    b -= W.wb[k] * W.mu[k] / W.sd[k];
  }
  out[d] = b;
}

int lr_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(1024, (n + 255) / 256)); }

LrWs carve_lr(void* ws, int64_t n, int d) {
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  LrWs W;
  W.counter = reinterpret_cast<unsigned*>(take(16));
  W.bad = W.counter + 1;
  W.cls = reinterpret_cast<double*>(take(16));
  W.mu = reinterpret_cast<double*>(take((size_t)d * 8));
  W.sd = reinterpret_cast<double*>(take((size_t)d * 8));
  W.wb = reinterpret_cast<double*>(take((size_t)(d + 1) * 8));
  W.part = reinterpret_cast<double*>(take((size_t)lr_blocks(n) * (d + 1) * 8));
  W.X = reinterpret_cast<double*>(take((size_t)n * d * 8));
  return W;
}
}  // namespace

size_t fit_ws_bytes(int64_t n, int32_t d, int64_t small_bytes) {
  const size_t ref = 256 + (size_t)((small_bytes + 15) / 16) * 16 * 8;
  const size_t lr = 16 * 256 + (size_t)d * 16 + (size_t)(d + 1) * 8 + (size_t)lr_blocks(n) * (d + 1) * 8 +
                    (size_t)n * d * 8 + 7 * 256;
  return std::max(ref, lr);
}

noscope_status launch_reference_image(const uint8_t* small, int64_t pitch, int bytes, const uint8_t* labels,
                                      int64_t n, uint8_t* ref, void* ws, uint64_t* neg_count_host,
                                      cudaStream_t st) {
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  unsigned long long* count = reinterpret_cast<unsigned long long*>(p);
  unsigned long long* sums = reinterpret_cast<unsigned long long*>(p + 256);
  const int nvec = (bytes + 15) / 16;
  NS_CUDA_TRY(cudaMemsetAsync(p, 0, 256 + (size_t)nvec * 16 * 8, st));
  // <= 2^32 / 255 frames per CTA keeps the u32 register sums exact
  const int64_t min_blocks = (n + 16000000 - 1) / 16000000;
  const int grid = (int)std::max<int64_t>(min_blocks, std::min<int64_t>(2 * kNumSMs, (n + 63) / 64));
  const int threads = nvec <= 512 ? ((nvec + 31) / 32) * 32 : 512;   // one pass when a frame fits
  ref_sum_kernel<<<std::max(grid, 1), threads, 0, st>>>(small, pitch, nvec, labels, n, sums, count);
  NS_LAUNCH_CHECK();
  ref_finish_kernel<<<(bytes + 255) / 256, 256, 0, st>>>(sums, count, bytes, ref);
  NS_LAUNCH_CHECK();
  count_launch(2);
  unsigned long long m = 0;
  NS_CUDA_TRY(cudaMemcpyAsync(&m, count, 8, cudaMemcpyDeviceToHost, st));
  NS_CUDA_TRY(cudaStreamSynchronize(st));
  *neg_count_host = m;
  return NOSCOPE_OK;
}

noscope_status launch_block_features(const noscope_dd_config& c, const uint8_t* small, int64_t pitch,
                                     int64_t n, double* feats, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(n, 8 * kNumSMs));
  block_feat_kernel<<<grid, kFitThreads, 0, st>>>(small, pitch, c.out_w, c.out_h, c.grid, c.mode,
                                                  c.ref_image, c.t_diff_frames, n, feats);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

noscope_status launch_lr_fit(const double* F, const uint8_t* t, int64_t n, int d, int iters, double lr,
                             double l2, double* wb_host, void* ws, cudaStream_t st) {
  LrWs W = carve_lr(ws, n, d);
  NS_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 16, st));
  NS_CUDA_TRY(cudaMemsetAsync(W.wb, 0, (size_t)(d + 1) * 8, st));
  const int nblk = lr_blocks(n);
  lr_stats_kernel<<<nblk, kFitThreads, 0, st>>>(F, t, n, d, 0, W);
  NS_LAUNCH_CHECK();
  lr_stats_kernel<<<nblk, kFitThreads, 0, st>>>(F, t, n, d, 1, W);
  NS_LAUNCH_CHECK();
  // check the inputs before iterating: one class only / non-finite features
  double cls = 0.0;
  unsigned bad = 0;
  NS_CUDA_TRY(cudaMemcpyAsync(&cls, W.cls, 8, cudaMemcpyDeviceToHost, st));
  NS_CUDA_TRY(cudaMemcpyAsync(&bad, W.bad, 4, cudaMemcpyDeviceToHost, st));
  NS_CUDA_TRY(cudaStreamSynchronize(st));
  count_launch(2);
  if (bad || cls < 1.0 || cls > (double)n - 1.0) return NOSCOPE_DATA;
  lr_standardize_kernel<<<(int)std::min<int64_t>((n * d + 255) / 256, 8 * kNumSMs), 256, 0, st>>>(F, n, d, W);
  NS_LAUNCH_CHECK();
  count_launch();
  if (lr <= 0.0) lr = 4.0 / (d + 1);
  const int64_t per = (n + nblk - 1) / nblk;
  const int P = std::max(1, kFitThreads / (d + 1));
  const size_t smem = (size_t)(d + 1 + per + (size_t)P * (d + 1)) * 8;
  constexpr size_t kMaxDyn = 220 * 1024;   // + the kernel's static shared flag
  static bool attr = false;
  if (!attr) {
    NS_CUDA_TRY(cudaFuncSetAttribute(lr_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDyn));
    attr = true;
  }
  if (smem > kMaxDyn) return NOSCOPE_SHAPE;
  for (int it = 0; it < iters; ++it) {
    lr_step_kernel<<<nblk, kFitThreads, smem, st>>>(t, n, d, per, lr, l2, W);
    NS_LAUNCH_CHECK();
  }
  count_launch(iters);
  double* out = W.part;   // reuse: d + 1 doubles
  lr_unscale_kernel<<<1, 32, 0, st>>>(d, W, out);
  NS_LAUNCH_CHECK();
  count_launch();
  NS_CUDA_TRY(cudaMemcpyAsync(wb_host, out, (size_t)(d + 1) * 8, cudaMemcpyDeviceToHost, st));
  NS_CUDA_TRY(cudaStreamSynchronize(st));
  return NOSCOPE_OK;
}

}  // namespace ns
