// fit.cu — the difference detector's fitting steps on the
// GPU: the reference image ("computes the reference image by averaging
// frames where the reference model returns no labels"), per-frame block-MSE
// features, and the blocked-LR weights ("trains a logistic regression
// (LR) classifier to weigh each block").  Readings R-21 / R-22
// (DESIGN.md): half-up rounding of the mean on the 50x50 small frames; LR = the
// minimiser of the l2-regularised mean log loss on z-scored features (Newton).
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
// Reading R-22: the minimiser of J(w, b) = mean_i[softplus(z_i) - t_i z_i] +
// l2/2 |w|^2 over z-scored features, by Newton's method with Armijo backtracking
// over the step ladder 1, 1/2, ..., 2^-15, to max|grad J| <= tol.  Per iteration:
//   lr_grad_hess_kernel   per-CTA partials of X1^T r, X1^T S X1 (upper triangle)
//                         and the loss over a fixed row range
//   lr_newton_kernel      (1 CTA) partials summed in CTA order -> g, H, J; stop
//                         test; Cholesky of H, Delta = -H^{-1} g, slope g.Delta
//   lr_trial_kernel       per-CTA loss partials at all 16 trial steps in one pass
//   lr_accept_kernel      (1 CTA) first step meeting Armijo; v += s Delta
constexpr int kLrSteps = 16;
constexpr int kLrRows = 32;          // rows staged per chunk in lr_grad_hess_kernel
constexpr int kLrSolveThreads = 1024;
constexpr int kLrMaxD = 256;         // grid <= 16

struct LrWs {
  double* X;          // [d][n] z-scored features (column-major: coalesced rows)
  double* mu;         // [d]
  double* sd;         // [d]
  double* part;       // [nblk][E*E + E + 1] per-CTA partials (H upper, g, loss); stats use [nblk][E]
  double* part_ls;    // [nblk][kLrSteps] trial-loss partials
  double* H;          // [E][E] Hessian, factored in place (lower triangle = L)
  double* wb;         // [E] parameters (w..., b)
  double* g;          // [E] gradient at wb
  double* delta;      // [E] Newton direction
  double* scal;       // [0] J(wb)  [1] g.delta  [2] max|g|  [3] accepted steps
  unsigned* counter;  // last-CTA arrival counter (stats)
  unsigned* bad;      // non-finite feature / target flag
  unsigned* done;     // 0 running, 1 converged, 2 no Armijo step, 3 max iterations, 4 H not PD
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

__device__ __forceinline__ double softplus_minus(double z, double t) {
  // log(1 + e^z) - t z, overflow-free
  return fmax(z, 0.0) + log1p(exp(-fabs(z))) - t * z;
}

__global__ void __launch_bounds__(kFitThreads)
lr_grad_hess_kernel(const uint8_t* __restrict__ t, int64_t n, int d, int64_t per, LrWs W) {
  if (*W.done) return;
  extern __shared__ double sh[];
  const int E = d + 1;
  double* w = sh;                         // [E]
  double* xs = w + E;                     // [kLrRows][E]
  double* rs = xs + kLrRows * E;          // [kLrRows]
  double* ss = rs + kLrRows;              // [kLrRows]
  double* ls = ss + kLrRows;              // [kLrRows] per-row-slot loss sums
  const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  const int PL = E * E + E;
  double* part = W.part + (size_t)blockIdx.x * (PL + 1);
  for (int k = threadIdx.x; k < E; k += blockDim.x) w[k] = W.wb[k];
  for (int e = threadIdx.x; e < PL; e += blockDim.x) part[e] = 0.0;
  if (threadIdx.x < kLrRows) ls[threadIdx.x] = 0.0;
  __syncthreads();
  for (int64_t c0 = r0; c0 < r1; c0 += kLrRows) {
    for (int e = threadIdx.x; e < kLrRows * E; e += blockDim.x) {
      const int i = e % kLrRows, k = e / kLrRows;
      const int64_t row = c0 + i;
      xs[i * E + k] = row < r1 ? (k < d ? W.X[(size_t)k * n + row] : 1.0) : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < kLrRows) {
      const int i = threadIdx.x;
      if (c0 + i < r1) {
        double z = w[d];
        for (int k = 0; k < d; ++k) z += xs[i * E + k] * w[k];
        const double p = 1.0 / (1.0 + exp(-z));
        const double ti = (double)(t[c0 + i] != 0);
        rs[i] = p - ti;
        ss[i] = p * (1.0 - p);
        ls[i] += softplus_minus(z, ti);
      } else {
        rs[i] = 0.0;
        ss[i] = 0.0;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < PL; e += blockDim.x) {
      double acc = 0.0;
      if (e < E * E) {
        const int k = e / E, l = e - k * E;
        if (l < k) continue;
        for (int i = 0; i < kLrRows; ++i) acc += xs[i * E + k] * xs[i * E + l] * ss[i];
      } else {
        const int k = e - E * E;
        for (int i = 0; i < kLrRows; ++i) acc += xs[i * E + k] * rs[i];
      }
      part[e] += acc;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double L = 0.0;
    for (int i = 0; i < kLrRows; ++i) L += ls[i];
    part[PL] = L;
  }
}

__global__ void __launch_bounds__(kLrSolveThreads)
lr_newton_kernel(int64_t n, int d, int nblk, double l2, double tol, int it, int max_iters, LrWs W) {
  __shared__ double red[kLrSolveThreads / 32];
  __shared__ int status;
  const int E = d + 1, PL = E * E + E;
  if (threadIdx.x == 0) status = (int)*W.done;
  __syncthreads();
  if (status) return;
  // partials summed in CTA order: H (mirrored), g, J
  for (int e = threadIdx.x; e <= PL; e += blockDim.x) {
    int k = 0, l = 0;
    if (e < E * E) {
      k = e / E;
      l = e - k * E;
      if (l < k) continue;
    }
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += W.part[(size_t)b * (PL + 1) + e];
    s /= (double)n;
    if (e < E * E) {
      if (k == l && k < d) s += l2;
      W.H[k * E + l] = s;
      W.H[l * E + k] = s;
    } else if (e < PL) {
      const int q = e - E * E;
      W.g[q] = s + (q < d ? l2 * W.wb[q] : 0.0);
    } else {
      W.scal[0] = s;            // mean loss; the penalty is added below
    }
  }
  __syncthreads();
  double m = 0.0;
  for (int k = threadIdx.x; k < E; k += blockDim.x) m = fmax(m, fabs(W.g[k]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0, ww = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) g = fmax(g, red[i]);
    for (int k = 0; k < d; ++k) ww += W.wb[k] * W.wb[k];
    W.scal[0] += 0.5 * l2 * ww;
    W.scal[2] = g;
    status = g <= tol ? 1 : (it >= max_iters ? 3 : 0);
    if (status) *W.done = (unsigned)status;
  }
  __syncthreads();
  if (status) return;
  // Cholesky H = L L^T in place (lower triangle), right-looking, one column per step
  double* H = W.H;
  for (int j = 0; j < E; ++j) {
    if (threadIdx.x == 0) {
      const double a = H[j * E + j];
      if (!(a > 0.0)) {
        status = 4;
        *W.done = 4u;
      } else {
        H[j * E + j] = sqrt(a);
      }
    }
    __syncthreads();
    if (status) return;
    const double ljj = H[j * E + j];
    for (int i = j + 1 + threadIdx.x; i < E; i += blockDim.x) H[i * E + j] /= ljj;
    __syncthreads();
    const int m2 = E - j - 1;
    for (int e = threadIdx.x; e < m2 * m2; e += blockDim.x) {
      const int i = j + 1 + e / m2, k = j + 1 + e % m2;
      if (k <= i) H[i * E + k] -= H[i * E + j] * H[k * E + j];
    }
    __syncthreads();
  }
  // L y = -g (forward), L^T delta = y (backward); y and delta in W.delta
  double* y = W.delta;
  for (int k = threadIdx.x; k < E; k += blockDim.x) y[k] = -W.g[k];
  __syncthreads();
  for (int j = 0; j < E; ++j) {
    if (threadIdx.x == 0) y[j] /= H[j * E + j];
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < E; i += blockDim.x) y[i] -= H[i * E + j] * y[j];
    __syncthreads();
  }
  for (int j = E - 1; j >= 0; --j) {
    if (threadIdx.x == 0) y[j] /= H[j * E + j];
    __syncthreads();
    for (int i = threadIdx.x; i < j; i += blockDim.x) y[i] -= H[j * E + i] * y[j];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double sl = 0.0;
    for (int k = 0; k < E; ++k) sl += W.g[k] * y[k];
    W.scal[1] = sl;
  }
}

__global__ void __launch_bounds__(kFitThreads)
lr_trial_kernel(const uint8_t* __restrict__ t, int64_t n, int d, int64_t per, LrWs W) {
  if (*W.done) return;
  __shared__ double red[kFitThreads][kLrSteps + 1];
  const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  double acc[kLrSteps];
#pragma unroll
  for (int q = 0; q < kLrSteps; ++q) acc[q] = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double z0 = W.wb[d], dz = W.delta[d];
    for (int k = 0; k < d; ++k) {
      const double x = W.X[(size_t)k * n + i];
      z0 += x * W.wb[k];
      dz += x * W.delta[k];
    }
    const double ti = (double)(t[i] != 0);
    double s = 1.0;
#pragma unroll
    for (int q = 0; q < kLrSteps; ++q, s *= 0.5) acc[q] += softplus_minus(z0 + s * dz, ti);
  }
#pragma unroll
  for (int q = 0; q < kLrSteps; ++q) red[threadIdx.x][q] = acc[q];
  __syncthreads();
  if (threadIdx.x < kLrSteps) {
    double s = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) s += red[i][threadIdx.x];
    W.part_ls[(size_t)blockIdx.x * kLrSteps + threadIdx.x] = s;
  }
}

__global__ void lr_accept_kernel(int64_t n, int d, int nblk, double l2, LrWs W) {
  __shared__ double Js[kLrSteps];
  __shared__ int pick;
  if (*W.done) return;
  const int E = d + 1;
  if (threadIdx.x < kLrSteps) {
    const double s = ldexp(1.0, -(int)threadIdx.x);
    double L = 0.0;
    for (int b = 0; b < nblk; ++b) L += W.part_ls[(size_t)b * kLrSteps + threadIdx.x];
    double ww = 0.0;
    for (int k = 0; k < d; ++k) {
      const double v = W.wb[k] + s * W.delta[k];
      ww += v * v;
    }
    Js[threadIdx.x] = L / (double)n + 0.5 * l2 * ww;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pick = -1;
    for (int q = 0; q < kLrSteps; ++q) {
      const double s = ldexp(1.0, -q);
      if (Js[q] <= W.scal[0] + 1e-4 * s * W.scal[1]) {
        pick = q;
        break;
      }
    }
    if (pick < 0) *W.done = 2u;
    else W.scal[3] += 1.0;
  }
  __syncthreads();
  if (pick < 0) return;
  const double s = ldexp(1.0, -pick);
  for (int k = threadIdx.x; k < E; k += blockDim.x) W.wb[k] += s * W.delta[k];
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

int lr_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, (n + 255) / 256)); }
size_t lr_part_doubles(int64_t n, int d) {
  const size_t E = (size_t)d + 1;
  return (size_t)lr_blocks(n) * (E * E + E + 1);
}

LrWs carve_lr(void* ws, int64_t n, int d) {
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  LrWs W;
  const size_t E = (size_t)d + 1;
  W.counter = reinterpret_cast<unsigned*>(take(16));
  W.bad = W.counter + 1;
  W.done = W.counter + 2;
  W.cls = reinterpret_cast<double*>(take(16));
  W.scal = reinterpret_cast<double*>(take(4 * 8));
  W.mu = reinterpret_cast<double*>(take((size_t)d * 8));
  W.sd = reinterpret_cast<double*>(take((size_t)d * 8));
  W.wb = reinterpret_cast<double*>(take(E * 8));
  W.g = reinterpret_cast<double*>(take(E * 8));
  W.delta = reinterpret_cast<double*>(take(E * 8));
  W.H = reinterpret_cast<double*>(take(E * E * 8));
  W.part_ls = reinterpret_cast<double*>(take((size_t)lr_blocks(n) * kLrSteps * 8));
  W.part = reinterpret_cast<double*>(take(lr_part_doubles(n, d) * 8));
  W.X = reinterpret_cast<double*>(take((size_t)n * d * 8));
  return W;
}
}  // namespace

size_t fit_ws_bytes(int64_t n, int32_t d, int64_t small_bytes) {
  const size_t ref = 256 + (size_t)((small_bytes + 15) / 16) * 16 * 8;
  const size_t E = (size_t)d + 1;
  const size_t lr = 16 * 256 + 256 + (size_t)d * 16 + 3 * E * 8 + E * E * 8 +
                    (size_t)lr_blocks(n) * kLrSteps * 8 + lr_part_doubles(n, d) * 8 + (size_t)n * d * 8 + 12 * 256;
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

noscope_status launch_lr_fit(const double* F, const uint8_t* t, int64_t n, int d, int max_iters, double tol,
                             double l2, double* wb_host, double* info_host, void* ws, cudaStream_t st) {
  if (d > kLrMaxD) return NOSCOPE_SHAPE;
  LrWs W = carve_lr(ws, n, d);
  NS_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 16, st));
  NS_CUDA_TRY(cudaMemsetAsync(W.scal, 0, 4 * 8, st));
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
  const int64_t per = (n + nblk - 1) / nblk;
  const int E = d + 1;
  const size_t smem = (size_t)(E + kLrRows * E + 3 * kLrRows) * 8;
  // set on every call: function attributes are per device context
  NS_CUDA_TRY(cudaFuncSetAttribute(lr_grad_hess_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned done = 0;
  for (int it = 0;; ++it) {
    lr_grad_hess_kernel<<<nblk, kFitThreads, smem, st>>>(t, n, d, per, W);
    NS_LAUNCH_CHECK();
    lr_newton_kernel<<<1, kLrSolveThreads, 0, st>>>(n, d, nblk, l2, tol, it, max_iters, W);
    NS_LAUNCH_CHECK();
    count_launch(2);
    NS_CUDA_TRY(cudaMemcpyAsync(&done, W.done, 4, cudaMemcpyDeviceToHost, st));
    NS_CUDA_TRY(cudaStreamSynchronize(st));
    if (done) break;
    lr_trial_kernel<<<nblk, kFitThreads, 0, st>>>(t, n, d, per, W);
    NS_LAUNCH_CHECK();
    lr_accept_kernel<<<1, 32, 0, st>>>(n, d, nblk, l2, W);
    NS_LAUNCH_CHECK();
    count_launch(2);
  }
  if (done == 4u) return NOSCOPE_DATA;
  double* out = W.part_ls;   // reuse: d + 1 doubles
  lr_unscale_kernel<<<1, 32, 0, st>>>(d, W, out);
  NS_LAUNCH_CHECK();
  count_launch();
  NS_CUDA_TRY(cudaMemcpyAsync(wb_host, out, (size_t)(d + 1) * 8, cudaMemcpyDeviceToHost, st));
  double sc[4];
  NS_CUDA_TRY(cudaMemcpyAsync(sc, W.scal, 4 * 8, cudaMemcpyDeviceToHost, st));
  NS_CUDA_TRY(cudaStreamSynchronize(st));
  if (info_host) {
    info_host[0] = sc[3];          // accepted Newton steps
    info_host[1] = sc[2];          // max|grad J| at the returned point
    info_host[2] = sc[0];          // J at the returned point
    info_host[3] = (double)done;   // 1 tol met, 2 no Armijo step (rounding floor), 3 max_iters
  }
  return NOSCOPE_OK;
}

}  // namespace ns
