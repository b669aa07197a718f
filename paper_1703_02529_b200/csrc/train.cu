// train.cu — specialized-CNN training on the GPU (P:472-477
// "RMSprop ... between one and five epochs ... early stopping"
// cross-validation).  Reading R-25: fp32 forward/backward without
// bf16 rounding (input = the inference normalisation), mean binary cross-entropy
// on the logit, RMSprop, max-pool gradient to the first maximum of each window.
//
// Every convolution and dense layer is a GEMM on explicit im2col rows, run on
// the tcgen05 tensor cores at fp32 accuracy (gemm_tc.cu, 3xTF32: forward
// Y = cols W^T, weight gradient dW = dY^T cols, input gradient dcols = dY W, bias
// gradients = dY^T 1); the kernels here do the rest: normalisation + gather,
// im2col / col2im (gather form, no atomics), bias + ReLU + 2x2 max pool with
// argmax, the unpool/ReLU mask, the dense-head elementwise steps, the loss and
// RMSprop.  No atomics anywhere (split-K partials are summed in a fixed order),
// so a run is reproducible.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace ns {

namespace {
constexpr int kT = 256;
#define NS_TRY(expr)                          \
  do {                                        \
    noscope_status _s = (expr);               \
    if (_s != NOSCOPE_OK) return _s;          \
  } while (0)

inline int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 16 * kNumSMs)); }

// x = bf16_RNE(clamp(((float)g - mu) / 127.5f, -1, 1)) (the inference input), NHWC fp32
__global__ void norm_gather_kernel(const uint8_t* __restrict__ small, int64_t pitch, const int32_t* __restrict__ idx,
                                   int B, float m0, float m1, float m2, float* __restrict__ x) {
  const int64_t total = (int64_t)B * 7500;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / 7500), r = (int)(e % 7500), c = r % 3;
    const float g = (float)small[(int64_t)idx[b] * pitch + r];
    const float mu = c == 0 ? m0 : (c == 1 ? m1 : m2);
    const float v = fminf(fmaxf((g - mu) / 127.5f, -1.0f), 1.0f);
    x[e] = __bfloat162float(__float2bfloat16_rn(v));
  }
}

// cols[(b*H + y)*W + x][(ky*3 + kx)*C + c] = x[b][y+ky-1][x+kx-1][c] (0 outside).
// One thread per (pixel, tap, 4-channel group) when C % 4 == 0 (float4 copies),
// else per (pixel, tap) copying C scalars: the index arithmetic is paid once.
__global__ void im2col_kernel(const float* __restrict__ x, int B, int H, int W, int C, float* __restrict__ cols) {
  const int K = 9 * C;
  const int vec = (C % 4 == 0) ? C / 4 : 1;
  const int64_t total = (int64_t)B * H * W * 9 * vec;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(e % vec);
    const int64_t pt = e / vec;
    const int tap = (int)(pt % 9);
    const int64_t p = pt / 9;
    const int xx = (int)(p % W);
    const int64_t by = p / W;
    const int yy = (int)(by % H);
    const int sy = yy + tap / 3 - 1, sx = xx + tap % 3 - 1;
    const bool in = sy >= 0 && sy < H && sx >= 0 && sx < W;
    float* dst = cols + p * K + tap * C;
    const float* src = x + (p + (int64_t)(sy - yy) * W + (sx - xx)) * C;
    if (C % 4 == 0) {
      reinterpret_cast<float4*>(dst)[v] = in ? reinterpret_cast<const float4*>(src)[v] : make_float4(0, 0, 0, 0);
    } else {
      for (int c = 0; c < C; ++c) dst[c] = in ? src[c] : 0.0f;
    }
  }
}

// a = relu(pre + bias) for the pooled region (in place), pooled = 2x2 max,
// arg = first maximum in (dy, dx) order.  Rows/columns outside the floor pool
// region are set to 0 (they never receive a gradient).
__global__ void bias_relu_pool_kernel(float* __restrict__ a, const float* __restrict__ bias, int B, int H, int W,
                                      int C, float* __restrict__ pooled, uint8_t* __restrict__ arg) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)B * Ho * Wo * C;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    const int64_t q = e / C;
    const int xo = (int)(q % Wo), yo = (int)((q / Wo) % Ho);
    const int64_t b = q / ((int64_t)Wo * Ho);
    float best = 0.0f;
    int bi = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int64_t off = ((b * H + 2 * yo + (m >> 1)) * W + 2 * xo + (m & 1)) * C + c;
      const float v = fmaxf(a[off] + bias[c], 0.0f);
      a[off] = v;
      if (m == 0 || v > best) { best = v; bi = m; }
    }
    pooled[e] = best;
    arg[e] = (uint8_t)bi;
  }
  // the row / column dropped by the floor pool (odd H, W)
  if ((H & 1) || (W & 1)) {
    const int64_t edge = (int64_t)B * (H * W - 4 * Ho * Wo) * C;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < edge; e += (int64_t)gridDim.x * blockDim.x) {
      const int c = (int)(e % C);
      const int64_t q = e / C;
      const int per = H * W - 4 * Ho * Wo;
      const int64_t b = q / per;
      const int r = (int)(q % per);
      int y, x;
      if (r < W * (H - 2 * Ho)) { y = 2 * Ho + r / W; x = r % W; }
      else { const int s = r - W * (H - 2 * Ho); y = s / (W - 2 * Wo); x = 2 * Wo + s % (W - 2 * Wo); }
      a[((b * H + y) * W + x) * C + c] = 0.0f;
    }
  }
}

// da (in place over a): the pooled gradient goes to the window's argmax if its
// activation is positive (ReLU'), every other position gets 0
__global__ void unpool_relu_kernel(float* __restrict__ a, const float* __restrict__ dpooled,
                                   const uint8_t* __restrict__ arg, int B, int H, int W, int C) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)B * Ho * Wo * C;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    const int64_t q = e / C;
    const int xo = (int)(q % Wo), yo = (int)((q / Wo) % Ho);
    const int64_t b = q / ((int64_t)Wo * Ho);
    const int am = arg[e];
    const float g = dpooled[e];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int64_t off = ((b * H + 2 * yo + (m >> 1)) * W + 2 * xo + (m & 1)) * C + c;
      a[off] = (m == am && a[off] > 0.0f) ? g : 0.0f;
    }
  }
}

// dx[b][y][x][c] = sum_{ky,kx} dcols[(b, y-ky+1, x-kx+1)][(ky*3+kx)*C + c] (gather)
__global__ void col2im_kernel(const float* __restrict__ dcols, int B, int H, int W, int C, float* __restrict__ dx) {
  const int K = 9 * C;
  const int64_t total = (int64_t)B * H * W * C;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    const int64_t p = e / C;
    const int xx = (int)(p % W), yy = (int)((p / W) % H);
    const int64_t b = p / ((int64_t)W * H);
    float s = 0.0f;
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int oy = yy - ky + 1, ox = xx - kx + 1;
        if (oy >= 0 && oy < H && ox >= 0 && ox < W)
          s += dcols[((b * H + oy) * W + ox) * K + (ky * 3 + kx) * C + c];
      }
    dx[e] = s;
  }
}

__global__ void bias_relu_kernel(float* __restrict__ h, const float* __restrict__ bias, int B, int D) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < B * D; e += gridDim.x * blockDim.x)
    h[e] = fmaxf(h[e] + bias[e % D], 0.0f);
}

// z = h1 . w2 + b2; loss partial (fixed order, one block); dz = (sigmoid(z) - t) / B
__global__ void head_kernel(const float* __restrict__ h1, const float* __restrict__ w2, const float* __restrict__ b2,
                            const uint8_t* __restrict__ labels, const int32_t* __restrict__ idx, int B, int D,
                            float* __restrict__ dz, double* __restrict__ loss_acc, int want_grad) {
  __shared__ double red[kT];
  double l = 0.0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    float z = b2[0];
    for (int d = 0; d < D; ++d) z = fmaf(h1[b * D + d], w2[d], z);
    const float t = labels[idx[b]] ? 1.0f : 0.0f;
    // softplus(z) - t z, stable: max(z, 0) + log1p(exp(-|z|)) - t z
    l += (double)(fmaxf(z, 0.0f) + log1pf(expf(-fabsf(z))) - t * z);
    if (want_grad) dz[b] = (1.0f / (1.0f + expf(-z)) - t) / (float)B;
  }
  red[threadIdx.x] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < blockDim.x; ++i) s += red[i];
    *loss_acc += s;
  }
}

// g_w2[d] = sum_b h1[b][d] dz[b]; g_b2 = sum_b dz[b]; dh1 = dz w2 (h1 > 0)
__global__ void head_grad_kernel(const float* __restrict__ h1, const float* __restrict__ w2, const float* __restrict__ dz,
                                 int B, int D, float* __restrict__ g_w2, float* __restrict__ g_b2,
                                 float* __restrict__ dh1) {
  for (int d = threadIdx.x; d <= D; d += blockDim.x) {
    float s = 0.0f;
    for (int b = 0; b < B; ++b) s += d < D ? h1[b * D + d] * dz[b] : dz[b];
    if (d < D) g_w2[d] = s;
    else g_b2[0] = s;
  }
  for (int e = threadIdx.x; e < B * D; e += blockDim.x)
    dh1[e] = h1[e] > 0.0f ? dz[e / D] * w2[e % D] : 0.0f;
}

// Column sums out[c] = sum_r m[r][c] of a row-major [rows][C] matrix (the bias
// gradients), deterministic: block b sums the fixed row range [rows*b/nb, rows*(b+1)/nb)
// with per-thread partials in row order and a fixed smem fold, colsum_final_kernel adds
// the blocks' partials in block order.  C is a power of two <= 1024.
constexpr int kCsBlocks = 192;
__global__ void colsum_partial_kernel(const float* __restrict__ m, int64_t rows, int C, float* __restrict__ part) {
  extern __shared__ float red[];
  const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
  const int c = threadIdx.x % C, g = threadIdx.x / C, ng = blockDim.x / C;
  float acc = 0.0f;
  for (int64_t r = r0 + g; r < r1; r += ng) acc += m[r * C + c];
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < C) {
    float t = 0.0f;
    for (int k = 0; k < ng; ++k) t += red[k * C + threadIdx.x];
    part[(int64_t)blockIdx.x * C + threadIdx.x] = t;
  }
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int nb, int C, float* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    float t = 0.0f;
    for (int b = 0; b < nb; ++b) t += part[(int64_t)b * C + c];
    out[c] = t;
  }
}


__global__ void rmsprop_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ v, int64_t n,
                               float lr, float rho, float eps) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float gg = g[e];
    const float vv = rho * v[e] + (1.0f - rho) * gg * gg;
    v[e] = vv;
    p[e] -= lr * gg / (sqrtf(vv) + eps);
  }
}

// fp32 parameters -> inference weights (bf16 RNE conv / FC weights, fp32 biases)
__global__ void to_bf16_kernel(const float* __restrict__ s, uint16_t* __restrict__ d, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const __nv_bfloat16 h = __float2bfloat16_rn(s[e]);
    d[e] = *reinterpret_cast<const uint16_t*>(&h);
  }
}

// ---------------------------------------------------------------- host plan
struct TLayer { int H, W, cin, cout; int64_t w_off, b_off; };
struct TPlan {
  int L, D, K;
  TLayer lay[4];
  int64_t fc1_w, fc1_b, fc2_w, fc2_b, nparams;
};

TPlan make_tplan(const noscope_cnn_arch& a) {
  TPlan p{};
  p.L = a.n_conv;
  p.D = a.dense;
  int h = a.in_h, cin = 3;
  int64_t off = 0;
  for (int l = 0; l < p.L; ++l) {
    const int cout = a.base_filters << l;
    p.lay[l] = TLayer{h, h, cin, cout, off, off + (int64_t)cout * 9 * cin};
    off += (int64_t)cout * 9 * cin + cout;
    cin = cout;
    h /= 2;
  }
  p.K = h * h * cin;
  p.fc1_w = off;
  p.fc1_b = off + (int64_t)p.D * p.K;
  p.fc2_w = p.fc1_b + p.D;
  p.fc2_b = p.fc2_w + p.D;
  p.nparams = p.fc2_b + 1;
  return p;
}

// Row-major C[M][N] = op(A) op(B), op(A) M x K (transposes are strides, not copies).
noscope_status gemm_rm(bool ta, bool tb, int M, int N, int64_t K, const float* A, int64_t lda, const float* B,
                       int64_t ldb, float* C, int64_t ldc, float* part, cudaStream_t st) {
  return tc_gemm(A, ta ? 1 : lda, ta ? lda : 1, B, tb ? ldb : 1, tb ? 1 : ldb, C, ldc, M, N, K, part, st);
}

struct TWs {
  float *G, *V, *best, *x[5], *a[4], *cols[4], *dcols, *dx, *dxb, *h1, *dz, *dh1, *part, *cspart;
  uint8_t* arg[4];
  int32_t* idx_tmp;
  double* loss;
  size_t total;
};

TWs carve_t(const TPlan& p, int B, void* base) {
  uint8_t* c = reinterpret_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* r = c ? c + off : nullptr;
    off = (off + bytes + 255) & ~size_t(255);
    return r;
  };
  TWs w{};
  w.G = (float*)take(p.nparams * 4);
  w.V = (float*)take(p.nparams * 4);
  w.best = (float*)take(p.nparams * 4);
  size_t cols = 0, xmax = 0;
  for (int l = 0; l < p.L; ++l) {
    const TLayer& t = p.lay[l];
    w.x[l] = (float*)take((size_t)B * t.H * t.W * t.cin * 4);
    w.a[l] = (float*)take((size_t)B * t.H * t.W * t.cout * 4);
    w.arg[l] = take((size_t)B * (t.H / 2) * (t.W / 2) * t.cout);
    // each layer keeps its forward im2col rows for the weight gradient
    w.cols[l] = (float*)take((size_t)B * t.H * t.W * 9 * t.cin * 4);
    cols = std::max(cols, (size_t)B * t.H * t.W * 9 * t.cin);
    xmax = std::max(xmax, (size_t)B * t.H * t.W * t.cin);
    xmax = std::max(xmax, (size_t)B * (t.H / 2) * (t.W / 2) * t.cout);
  }
  w.x[p.L] = (float*)take((size_t)B * p.K * 4);
  w.dcols = (float*)take(cols * 4);
  w.dx = (float*)take(xmax * 4);
  w.dxb = (float*)take(xmax * 4);
  w.h1 = (float*)take((size_t)B * p.D * 4);
  w.dz = (float*)take((size_t)B * 4);
  w.dh1 = (float*)take((size_t)B * p.D * 4);
  // split-K scratch of the largest GEMM of a step (the weight gradients)
  size_t part = 0;
  auto need = [&](int M, int N, int64_t K) { part = std::max(part, tc_gemm_part_floats(M, N, K)); };
  for (int l = 0; l < p.L; ++l) {
    const TLayer& t = p.lay[l];
    const int64_t rows = (int64_t)B * t.H * t.W;
    need((int)rows, t.cout, 9 * t.cin);
    need(t.cout, 9 * t.cin, rows);
    need((int)rows, 9 * t.cin, t.cout);
  }
  need(B, p.D, p.K);
  need(p.D, p.K, B);
  need(B, p.K, p.D);
  w.part = (float*)take(std::max<size_t>(part, 1) * 4);
  w.loss = (double*)take(8);
  w.idx_tmp = (int32_t*)take((size_t)B * 4);   // the captured step's batch indices
  w.cspart = (float*)take((size_t)kCsBlocks * 1024 * 4);   // column-sum partials
  w.total = off;
  return w;
}

// column sums of a row-major [rows][C] matrix: out[c] = sum_r m[r][c] (the bias gradients;
// a dedicated reduction: as an N = 1 GEMM it cost a 32-wide tile and a split-K reduce)
noscope_status colsum(const float* m, int64_t rows, int C, float* out, float* part, cudaStream_t st) {
  const int threads = C <= 256 ? 256 : C;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(kCsBlocks, rows));
  colsum_partial_kernel<<<nb, threads, threads * sizeof(float), st>>>(m, rows, C, part);
  colsum_final_kernel<<<(C + 255) / 256, 256, 0, st>>>(part, nb, C, out);
  NS_LAUNCH_CHECK();
  return NOSCOPE_OK;
}

// Forward on B frames (idx on device); leaves activations for the backward pass,
// adds the batch's summed loss to *w.loss; dz if want_grad.
noscope_status forward(const TPlan& p, const noscope_cnn_arch& a, const float* P, TWs& w,
                       const uint8_t* small, int64_t pitch, const uint8_t* labels, const int32_t* idx, int B,
                       int want_grad, cudaStream_t st) {
  norm_gather_kernel<<<grid_for((int64_t)B * 7500), kT, 0, st>>>(small, pitch, idx, B, a.chan_mean[0],
                                                                  a.chan_mean[1], a.chan_mean[2], w.x[0]);
  for (int l = 0; l < p.L; ++l) {
    const TLayer& t = p.lay[l];
    const int64_t rows = (int64_t)B * t.H * t.W;
    im2col_kernel<<<grid_for(rows * 9 * (t.cin % 4 ? 1 : t.cin / 4)), kT, 0, st>>>(w.x[l], B, t.H, t.W, t.cin,
                                                                                 w.cols[l]);
    NS_TRY(gemm_rm(false, true, (int)rows, t.cout, 9 * t.cin, w.cols[l], 9 * t.cin, P + t.w_off, 9 * t.cin, w.a[l],
                   t.cout, w.part, st));
    bias_relu_pool_kernel<<<grid_for((int64_t)B * (t.H / 2) * (t.W / 2) * t.cout), kT, 0, st>>>(
        w.a[l], P + t.b_off, B, t.H, t.W, t.cout, w.x[l + 1], w.arg[l]);
  }
  NS_TRY(gemm_rm(false, true, B, p.D, p.K, w.x[p.L], p.K, P + p.fc1_w, p.K, w.h1, p.D, w.part, st));
  bias_relu_kernel<<<grid_for((int64_t)B * p.D), kT, 0, st>>>(w.h1, P + p.fc1_b, B, p.D);
  head_kernel<<<1, kT, 0, st>>>(w.h1, P + p.fc2_w, P + p.fc2_b, labels, idx, B, p.D, w.dz, w.loss, want_grad);
  NS_LAUNCH_CHECK();
  return NOSCOPE_OK;
}

noscope_status backward(const TPlan& p, const float* P, TWs& w, int B, cudaStream_t st) {
  float* G = w.G;
  head_grad_kernel<<<1, kT, 0, st>>>(w.h1, P + p.fc2_w, w.dz, B, p.D, G + p.fc2_w, G + p.fc2_b, w.dh1);
  NS_TRY(gemm_rm(true, false, p.D, p.K, B, w.dh1, p.D, w.x[p.L], p.K, G + p.fc1_w, p.K, w.part, st));
  NS_TRY(colsum(w.dh1, B, p.D, G + p.fc1_b, w.cspart, st));
  float* dpool = w.dx;   // gradient w.r.t. the current pooled map
  NS_TRY(gemm_rm(false, false, B, p.K, p.D, w.dh1, p.D, P + p.fc1_w, p.K, dpool, p.K, w.part, st));
  for (int l = p.L - 1; l >= 0; --l) {
    const TLayer& t = p.lay[l];
    const int64_t rows = (int64_t)B * t.H * t.W;
    unpool_relu_kernel<<<grid_for((int64_t)B * (t.H / 2) * (t.W / 2) * t.cout), kT, 0, st>>>(
        w.a[l], dpool, w.arg[l], B, t.H, t.W, t.cout);
    // dW = dY^T cols, on this layer's forward im2col rows
    NS_TRY(gemm_rm(true, false, t.cout, 9 * t.cin, rows, w.a[l], t.cout, w.cols[l], 9 * t.cin, G + t.w_off,
                   9 * t.cin, w.part, st));
    NS_TRY(colsum(w.a[l], rows, t.cout, G + t.b_off, w.cspart, st));
    if (l > 0) {
      NS_TRY(gemm_rm(false, false, (int)rows, 9 * t.cin, t.cout, w.a[l], t.cout, P + t.w_off, 9 * t.cin, w.dcols,
                     9 * t.cin, w.part, st));
      float* out = (dpool == w.dx) ? w.dxb : w.dx;
      col2im_kernel<<<grid_for(rows * t.cin), kT, 0, st>>>(w.dcols, B, t.H, t.W, t.cin, out);
      dpool = out;
    }
  }
  NS_LAUNCH_CHECK();
  return NOSCOPE_OK;
}
}  // namespace

int64_t train_param_count(const noscope_cnn_arch& a) { return make_tplan(a).nparams; }

size_t train_ws_bytes(const noscope_cnn_arch& a, int batch) {
  TPlan p = make_tplan(a);
  return carve_t(p, batch, nullptr).total + 256;
}

noscope_status launch_cnn_train(const noscope_cnn_arch& a, const noscope_train_config& cfg, float* P,
                                const uint8_t* small, int64_t pitch, const uint8_t* labels, const int32_t* perms,
                                int64_t n_train, const int32_t* val_idx, int64_t n_val, double* hist,
                                int32_t* epochs_run, void* ws, cudaStream_t st) {
  const TPlan p = make_tplan(a);
  TWs w = carve_t(p, cfg.batch, ws);
  noscope_status s = NOSCOPE_OK;
  // Full mini-batches replay one captured CUDA graph of the whole step (forward,
  // backward, RMSprop: ~40 dependent launches) with the batch's indices copied into
  // a fixed buffer first; the first batch (which also sets the kernels' attributes)
  // and a partial last batch run as plain launches.  Same kernels, same order: the
  // results are identical.  NOSCOPE_TRAIN_GRAPH=0 disables it (A/B).
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cs = nullptr;
  bool use_graph = true;
  if (const char* e = std::getenv("NOSCOPE_TRAIN_GRAPH")) use_graph = e[0] != '0';
  {
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cst) != cudaSuccess || cst != cudaStreamCaptureStatusNone) use_graph = false;
  }
  auto release = [&]() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (cs) cudaStreamDestroy(cs);
    gexec = nullptr;
    cs = nullptr;
  };
  auto fail = [&](noscope_status e) {
    release();
    return e;
  };
  auto step = [&](const int32_t* idx, int B, cudaStream_t s1) -> noscope_status {
    noscope_status r = forward(p, a, P, w, small, pitch, labels, idx, B, 1, s1);
    if (r != NOSCOPE_OK) return r;
    if ((r = backward(p, P, w, B, s1)) != NOSCOPE_OK) return r;
    rmsprop_kernel<<<grid_for(p.nparams), kT, 0, s1>>>(P, w.G, w.V, p.nparams, cfg.lr, cfg.rho, cfg.eps);
    NS_LAUNCH_CHECK();
    return NOSCOPE_OK;
  };
#define NS_TRAIN_TRY(expr)                                   \
  do {                                                       \
    if ((expr) != cudaSuccess) return fail(NOSCOPE_CUDA);    \
  } while (0)
  auto capture = [&]() -> noscope_status {
    cudaGraph_t g = nullptr;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return NOSCOPE_CUDA;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return NOSCOPE_CUDA;
    noscope_status r = step(w.idx_tmp, cfg.batch, cs);
    const cudaError_t ec = cudaStreamEndCapture(cs, &g);
    if (r != NOSCOPE_OK) return r;
    if (ec != cudaSuccess || !g) return NOSCOPE_CUDA;
    const cudaError_t ei = cudaGraphInstantiate(&gexec, g, 0);
    cudaGraphDestroy(g);
    return ei == cudaSuccess ? NOSCOPE_OK : NOSCOPE_CUDA;
  };
  NS_TRAIN_TRY(cudaMemsetAsync(w.V, 0, p.nparams * 4, st));
  NS_TRAIN_TRY(cudaMemcpyAsync(w.best, P, p.nparams * 4, cudaMemcpyDeviceToDevice, st));
  double best_val = INFINITY, prev_tr = INFINITY;
  int run = 0;
  for (int e = 0; e < cfg.epochs; ++e) {
    NS_TRAIN_TRY(cudaMemsetAsync(w.loss, 0, 8, st));
    for (int64_t s0 = 0; s0 < n_train; s0 += cfg.batch) {
      const int B = (int)std::min<int64_t>(cfg.batch, n_train - s0);
      const int32_t* idx = perms + (int64_t)e * n_train + s0;
      if (use_graph && B == cfg.batch && (e > 0 || s0 > 0)) {
        if (!gexec && (s = capture()) != NOSCOPE_OK) return fail(s);
        NS_TRAIN_TRY(cudaMemcpyAsync(w.idx_tmp, idx, (size_t)B * 4, cudaMemcpyDeviceToDevice, st));
        if (cudaGraphLaunch(gexec, st) != cudaSuccess) return fail(NOSCOPE_CUDA);
        continue;
      }
      if ((s = step(idx, B, st)) != NOSCOPE_OK) return fail(s);
    }
    double tr = 0.0, va = 0.0;
    NS_TRAIN_TRY(cudaMemcpyAsync(&tr, w.loss, 8, cudaMemcpyDeviceToHost, st));
    NS_TRAIN_TRY(cudaStreamSynchronize(st));
    NS_TRAIN_TRY(cudaMemsetAsync(w.loss, 0, 8, st));
    for (int64_t s0 = 0; s0 < n_val; s0 += cfg.batch) {
      const int B = (int)std::min<int64_t>(cfg.batch, n_val - s0);
      if ((s = forward(p, a, P, w, small, pitch, labels, val_idx + s0, B, 0, st)) != NOSCOPE_OK) return fail(s);
    }
    NS_TRAIN_TRY(cudaMemcpyAsync(&va, w.loss, 8, cudaMemcpyDeviceToHost, st));
    NS_TRAIN_TRY(cudaStreamSynchronize(st));
    tr /= (double)n_train;
    va /= (double)std::max<int64_t>(n_val, 1);
    hist[2 * e] = tr;
    hist[2 * e + 1] = va;
    run = e + 1;
    // keep the best cross-validation epoch; stop after the first epoch
    // whose training loss rose ("early stopping if the training loss
    // increases")
    if (va < best_val) {
      best_val = va;
      NS_TRAIN_TRY(cudaMemcpyAsync(w.best, P, p.nparams * 4, cudaMemcpyDeviceToDevice, st));
    }
    if (e > 0 && tr > prev_tr) break;
    prev_tr = tr;
  }
  NS_TRAIN_TRY(cudaMemcpyAsync(P, w.best, p.nparams * 4, cudaMemcpyDeviceToDevice, st));
  NS_TRAIN_TRY(cudaStreamSynchronize(st));
  release();
  *epochs_run = run;
  return NOSCOPE_OK;
}
#undef NS_TRAIN_TRY

noscope_status launch_params_to_weights(const noscope_cnn_arch& a, const float* P, const noscope_cnn_weights& wt,
                                        cudaStream_t st) {
  const TPlan p = make_tplan(a);
  for (int l = 0; l < p.L; ++l) {
    const TLayer& t = p.lay[l];
    const int64_t nw = (int64_t)t.cout * 9 * t.cin;
    to_bf16_kernel<<<grid_for(nw), kT, 0, st>>>(P + t.w_off, const_cast<uint16_t*>(wt.conv_w[l]), nw);
    NS_CUDA_TRY(cudaMemcpyAsync(const_cast<float*>(wt.conv_b[l]), P + t.b_off, t.cout * 4,
                                cudaMemcpyDeviceToDevice, st));
  }
  to_bf16_kernel<<<grid_for((int64_t)p.D * p.K), kT, 0, st>>>(P + p.fc1_w, const_cast<uint16_t*>(wt.fc1_w),
                                                              (int64_t)p.D * p.K);
  NS_CUDA_TRY(cudaMemcpyAsync(const_cast<float*>(wt.fc1_b), P + p.fc1_b, p.D * 4, cudaMemcpyDeviceToDevice, st));
  to_bf16_kernel<<<grid_for(p.D), kT, 0, st>>>(P + p.fc2_w, const_cast<uint16_t*>(wt.fc2_w), p.D);
  NS_CUDA_TRY(cudaMemcpyAsync(const_cast<float*>(wt.fc2_b), P + p.fc2_b, 4, cudaMemcpyDeviceToDevice, st));
  NS_LAUNCH_CHECK();
  return NOSCOPE_OK;
}

}  // namespace ns
