// cnn.cu — the specialized CNN (§4; north star: "3x3
// conv+ReLU+maxpool layers, a dense layer and a sigmoid") on tcgen05 tensor
// cores: bf16 operands from shared memory (or TMEM), fp32 accumulators in TMEM.
//
// Layer schedule per chunk of <= 32768 frames (kCnnChunk):
//   base_filters = 32: conv1+conv2 fused in one kernel (cnn_fused.cu; the conv1
//     map never leaves the SM), then conv3/conv4 (L = 4) on the generic layer
//     kernel (cnn_gemm.cu);
//   base_filters = 64: conv1 on the same fused kernel without the conv2 stage
//     (two N = 32 halves per A tile), its pooled map written to HBM in the
//     stacked layout, then conv2..convL on the generic layer kernel.
//   The last conv layer writes the FC feature tiles; fc_kernel does FC1 + ReLU
//   + FC2.
// FC: features (h, w, c) in the canonical A layout [tile][K/8][128][8] ->
//   tcgen05 GEMM with N = dense, epilogue bias+ReLU+bf16, FC2 dot + bias.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace ns {

constexpr int kCnnThreads = 128;
constexpr int kBStages = 4;
constexpr int64_t kCnnChunk = 32768;  // frames per internal chunk (workspace bound)
// L = 2 with conv2 fused: the only chunk-sized buffers are the FC features (K x 2 B per
// frame), so one chunk covers a whole webcam hour (no empty per-chunk launches when the
// device count is far below n_max)
constexpr int64_t kCnnChunkFusedL2 = 262144;

NS_DEV uint16_t f2bf(float v) {
  __nv_bfloat16 h = __float2bfloat16_rn(v);
  return *reinterpret_cast<uint16_t*>(&h);
}
NS_DEV float bf2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

static uint32_t tmem_cols_host(int c) {
  uint32_t r = 32;
  while ((int)r < c) r <<= 1;
  return r;
}


// ------------------------------------------------------------ weight packing
// out[((p*nkc + kc)*pn + n)*8 + e] = w[(p*pn + n)*Kreal + kc*8 + e] (0 beyond Kreal)


// =================================================================== FC
struct FcArgs {
  const uint8_t* feat;   // [tiles][K/8][128][8] bf16
  int K, D;
  const uint8_t* wpack;  // [K/8][D][8] bf16
  const float* b1;
  const uint16_t* w2;
  const float* b2;
  float* logits;
  const int64_t* n_dev;
  int64_t n_max, chunk_base, chunk_len;
  uint32_t tmem_cols;
  int ksplit;            // K split across CTAs (fixed per K: results do not depend on n)
  float* part;           // [tiles][ksplit][128][D] fp32 partial sums (ksplit > 1)
  unsigned* counters;    // [tiles] arrival counters, zero between uses
  const int32_t* fq;     // queue mode: row p is queue slot p, frame fq[p] ...
  const int32_t* pos_pf; // ... whose logit goes to logits[pos_pf[frame]] (null: index mode)
};
constexpr int kFcKChunk = 64;

// FC1 (+ReLU, bf16) and FC2 for one 128-frame tile and one K slice.  One
// CTA streams its features/weights through a kBStages bulk-copy ring; the K16
// steps alternate between two TMEM accumulators (independent MMA chains).
// With ksplit > 1 each CTA writes fp32 partials; the last CTA of a tile (arrival
// counter) sums them in slice order (deterministic) and runs the epilogue.
__global__ void __launch_bounds__(kCnnThreads)
fc_kernel(FcArgs A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int64_t n = min(*A.n_dev, A.n_max);
  const int64_t cnt = min(n - A.chunk_base, A.chunk_len);
  const int64_t tile = blockIdx.x / A.ksplit;
  const int ks = blockIdx.x % A.ksplit;
  if (cnt <= 0 || tile * 128 >= cnt) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t a_bytes = 128 * kFcKChunk * 2, b_bytes = (uint32_t)A.D * kFcKChunk * 2;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kBStages * stage_bytes);
  uint64_t* empty = full + kBStages;
  uint64_t* bar_acc = empty + kBStages;
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(bar_acc + 1);
  int* last = reinterpret_cast<int*>(tmem_s + 1);
  if (tid == 0) {
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(bar_acc, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_rt(tmem_s, A.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_s;
  const int nall = A.K / kFcKChunk;
  const int c0 = (int)((int64_t)nall * ks / A.ksplit), c1 = (int)((int64_t)nall * (ks + 1) / A.ksplit);
  const int nchunks = c1 - c0;
  const uint8_t* a_src = A.feat + tile * ((int64_t)A.K * 256) + (size_t)c0 * a_bytes;
  const uint8_t* b_src = A.wpack + (size_t)c0 * b_bytes;
  if (tid == 0) {
    auto issue = [&](int c) {
      const int s = c % kBStages;
      if (c >= kBStages) mbar_wait(&empty[s], (uint32_t)(((c / kBStages) - 1) & 1));
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      bulk_g2s(stages + (size_t)s * stage_bytes, a_src + (size_t)c * a_bytes, a_bytes, &full[s]);
      bulk_g2s(stages + (size_t)s * stage_bytes + a_bytes, b_src + (size_t)c * b_bytes, b_bytes,
               &full[s]);
    };
    int issued = 0;
    for (; issued < kBStages - 1 && issued < nchunks; ++issued) issue(issued);
    const uint32_t idesc = idesc_bf16_f32(128, A.D);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kBStages;
      mbar_wait(&full[s], (uint32_t)((c / kBStages) & 1));
      tc_fence_after();
      const uint32_t as = smem_u32(stages + (size_t)s * stage_bytes), bs = as + a_bytes;
#pragma unroll
      for (int kk = 0; kk < kFcKChunk / 16; ++kk)
        umma_bf16(tmem + (kk & 1) * A.D, sdesc(as + kk * 2 * 2048, 2048, 128),
                  sdesc(bs + kk * 2 * A.D * 16, A.D * 16, 128), idesc, (c > 0 || kk > 1) ? 1u : 0u);
      umma_commit(&empty[s]);
      if (issued < nchunks) issue(issued++);
    }
    umma_commit(bar_acc);
  }
  __syncwarp();
  mbar_wait(bar_acc, 0);
  tc_fence_after();
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  float* mypart = A.part + (((size_t)tile * A.ksplit + ks) * 128 + tid) * A.D;
  if (A.ksplit > 1) {
    for (int cb = 0; cb < A.D / 16; ++cb) {
      uint32_t r0[16], r1[16];
      tmem_ld16(trow + cb * 16, r0);
      tmem_ld16(trow + A.D + cb * 16, r1);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        *reinterpret_cast<float4*>(mypart + cb * 16 + j) =
            make_float4(__uint_as_float(r0[j]) + __uint_as_float(r1[j]),
                        __uint_as_float(r0[j + 1]) + __uint_as_float(r1[j + 1]),
                        __uint_as_float(r0[j + 2]) + __uint_as_float(r1[j + 2]),
                        __uint_as_float(r0[j + 3]) + __uint_as_float(r1[j + 3]));
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) *last = atomicAdd(&A.counters[tile], 1u) == (unsigned)(A.ksplit - 1);
    __syncthreads();
    if (!*last) {
      tc_fence_before();
      __syncthreads();
      if (warp == 0) tmem_dealloc_rt(tmem, A.tmem_cols);
      return;
    }
    __threadfence();
    if (tid == 0) A.counters[tile] = 0u;  // ready for the next chunk / call
  }
  float z = 0.0f;
  for (int cb = 0; cb < A.D / 16; ++cb) {
    float acc[16];
    if (A.ksplit > 1) {
      const float* p0 = A.part + ((size_t)tile * A.ksplit * 128 + tid) * A.D + cb * 16;
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0f;
      for (int k = 0; k < A.ksplit; ++k) {   // slice order: deterministic
        const float4* q = reinterpret_cast<const float4*>(p0 + (size_t)k * 128 * A.D);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 v = __ldcg(q + j);
          acc[4 * j] += v.x;
          acc[4 * j + 1] += v.y;
          acc[4 * j + 2] += v.z;
          acc[4 * j + 3] += v.w;
        }
      }
    } else {
      uint32_t r0[16], r1[16];
      tmem_ld16(trow + cb * 16, r0);
      tmem_ld16(trow + A.D + cb * 16, r1);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = __uint_as_float(r0[j]) + __uint_as_float(r1[j]);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = cb * 16 + j;
      const float h = bf2f(f2bf(fmaxf(acc[j] + A.b1[c], 0.0f)));
      z = fmaf(h, bf2f(A.w2[c]), z);
    }
  }
  z += A.b2[0];
  const int64_t row = tile * 128 + tid;
  if (row < cnt) A.logits[A.fq ? (int64_t)A.pos_pf[A.fq[row]] : A.chunk_base + row] = z;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc_rt(tmem, A.tmem_cols);
}

static int fc_ksplit(int K) { return std::max(1, std::min(4, K / 2304)); }

// =================================================================== host plan
struct CnnPlan {
  int L, C, D, K;
  bool fused;                 // conv2 fused into the conv1 kernel (base_filters = 32)
  int first_g;                // first layer on the generic kernel
  size_t w1_off, w2_off;      // fused: packed conv1 [4][32][8], conv2 [36][64][8]
  ConvGGeom g[4];             // generic layers first_g .. L-1
  size_t gw_off[4];           // their packed weights
  size_t in_off[4];           // their stacked inputs
  size_t fc_off, feat_off, part_off, cnt_off, total;
  int64_t chunk;
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// whole: one chunk of n_max frames (queue mode: features of every queue slot)
static bool make_plan(const noscope_cnn_arch& a, int64_t n_max, CnnPlan* P, bool whole = false) {
  CnnPlan p{};
  p.L = a.n_conv;
  p.C = a.base_filters;
  p.D = a.dense;
  p.fused = p.C == 32 || p.C == 16;
  p.first_g = p.fused ? 2 : 1;
  p.chunk = std::max<int64_t>(128, (n_max + 127) / 128 * 128);
  if (!whole) p.chunk = std::min<int64_t>(p.fused && p.L == 2 ? kCnnChunkFusedL2 : kCnnChunk, p.chunk);
  size_t off = 256;  // status words etc. live before the CNN region (caller offset)
  p.w1_off = off;
  off = align_up(off + (size_t)p.C * 32 * 2, 256);
  if (p.fused) {
    p.w2_off = off;
    off = align_up(off + (size_t)2 * p.C * 9 * p.C * 2, 256);
  }
  int h = 50, cin = 3;
  for (int l = 0; l < p.L; ++l) {
    const int cout = p.C << l;
    if (l >= p.first_g) {
      if (!make_convt_geom(cin, cout, h, p.chunk, &p.g[l]) &&
          !make_convg_geom(cin, cout, h, p.chunk, &p.g[l]))
        return false;
      p.gw_off[l] = off;
      off = align_up(off + (size_t)cout * p.g[l].steps * 32, 256);
    }
    cin = cout;
    h /= 2;
  }
  p.K = h * h * cin;
  if (p.K % kFcKChunk) return false;
  p.fc_off = off;
  off = align_up(off + (size_t)p.D * p.K * 2, 256);
  for (int l = p.first_g; l < p.L; ++l) {
    p.in_off[l] = off;
    off = align_up(off + (size_t)(p.g[l].cin_eff / 8) * p.g[l].R * 16, 1024);
  }
  p.feat_off = off;
  off = align_up(off + (size_t)p.chunk * p.K * 2, 1024);
  p.part_off = off;   // FC split-K partials
  off = align_up(off + (size_t)(p.chunk / 128) * fc_ksplit(p.K) * 128 * p.D * 4, 1024);
  p.cnt_off = off;
  off = align_up(off + (size_t)(p.chunk / 128) * 4, 256);
  p.total = off;
  *P = p;
  return true;
}

bool cnn_arch_supported(const noscope_cnn_arch& a) {
  if (a.in_w != 50 || a.in_h != 50) return false;
  if (a.n_conv != 2 && a.n_conv != 4) return false;
  if (a.base_filters != 16 && a.base_filters != 32 && a.base_filters != 64) return false;
  if (a.dense != 32 && a.dense != 64 && a.dense != 128 && a.dense != 256) return false;
  CnnPlan p;
  return make_plan(a, 128, &p);
}

size_t cnn_ws_bytes(const noscope_cnn_arch& a, int64_t n_max) {
  CnnPlan p;
  if (!make_plan(a, n_max, &p)) return 0;
  return p.total;
}

// Debug/test helper (see noscope_api.cu): per conv layer l the stacked input map
// {offset, rows per plane, H, channels (padded)} or -1, then the feature tiles.
bool cnn_debug_layout(const noscope_cnn_arch& a, int64_t n_max, int64_t* out) {
  CnnPlan p;
  if (!make_plan(a, n_max, &p)) return false;
  for (int l = 0; l < 4; ++l) {
    const bool g = l >= p.first_g && l < p.L;
    out[4 * l + 0] = g ? (int64_t)p.in_off[l] : -1;
    out[4 * l + 1] = g ? p.g[l].R : 0;
    out[4 * l + 2] = g ? p.g[l].H : 0;
    out[4 * l + 3] = g ? p.g[l].cin_eff : 0;
  }
  out[16] = (int64_t)p.feat_off;
  out[17] = p.K;
  out[18] = p.chunk;
  return true;
}

// All weight repacks of one call in ONE launch (the call is launch-latency bound
// for small batches): jobs share one flat index space; job 0 (conv1) also writes
// the fp32 bias as a bf16 hi/lo pair into K columns 27/28 (against A = 1.0).
struct PackJob {
  const uint16_t* w;
  uint16_t* out;
  int rows, Kreal, Kpad, pn;
  int64_t total;
};
struct PackJobs {
  PackJob j[3];
  int n;
  const float* bias1;  // conv1 bias (job 0), nullable
};
__global__ void pack_multi_kernel(PackJobs J) {
  int64_t start = 0;
  for (int q = 0; q < J.n; ++q) {
    const PackJob b = J.j[q];
    const int nkc = b.Kpad / 8;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - start; t < b.total;
         t += (int64_t)gridDim.x * blockDim.x) {
      if (t < 0) continue;
      const int e = (int)(t & 7);
      const int64_t r = t >> 3;
      const int n_all = (int)(r % b.rows);
      const int kc = (int)(r / b.rows);
      const int p = n_all / b.pn, n = n_all % b.pn;
      const int k = kc * 8 + e;
      uint16_t v = k < b.Kreal ? b.w[(int64_t)n_all * b.Kreal + k] : (uint16_t)0;
      if (q == 0 && J.bias1 && (k == 27 || k == 28)) {
        const float x = J.bias1[n_all];
        const __nv_bfloat16 hi = __float2bfloat16_rn(x);
        const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
        v = *reinterpret_cast<const uint16_t*>(k == 27 ? &hi : &lo);
      }
      b.out[(((int64_t)p * nkc + kc) * b.pn + n) * 8 + e] = v;
    }
    start += b.total;
  }
}


static noscope_status pack_weights(const CnnPlan& P, const noscope_cnn_weights& w, uint8_t* ws,
                                   cudaStream_t st) {
  PackJobs J{};
  auto job = [&](const uint16_t* wsrc, int rows, int Kreal, int Kpad, int pn, uint8_t* out) {
    J.j[J.n++] = PackJob{wsrc, reinterpret_cast<uint16_t*>(out), rows, Kreal, Kpad, pn,
                         (int64_t)rows * Kpad};
  };
  job(w.conv_w[0], P.C, 27, 32, P.C, ws + P.w1_off);  // + bias in K 27/28
  if (P.fused) job(w.conv_w[1], 2 * P.C, 9 * P.C, 9 * P.C, 2 * P.C, ws + P.w2_off);
  job(w.fc1_w, P.D, P.K, P.K, P.D, ws + P.fc_off);
  J.bias1 = w.conv_b[0];
  int64_t total = 0;
  for (int q = 0; q < J.n; ++q) total += J.j[q].total;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 4 * kNumSMs);
  pack_multi_kernel<<<grid, 256, 0, st>>>(J);
  NS_LAUNCH_CHECK();
  count_launch();
  for (int l = P.first_g; l < P.L; ++l) {
    noscope_status s = pack_convg(w.conv_w[l], P.g[l], ws + P.gw_off[l], st);
    if (s != NOSCOPE_OK) return s;
  }
  return NOSCOPE_OK;
}

static FusedArgs fused_args(const CnnPlan& P, const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                            const uint8_t* small, int64_t small_pitch, uint8_t* ws) {
  FusedArgs fa{};
  fa.C1 = P.C;
  fa.small = small;
  fa.small_pitch = small_pitch;
  fa.w1 = ws + P.w1_off;
  fa.w2 = P.fused ? ws + P.w2_off : nullptr;
  fa.b1 = w.conv_b[0];
  fa.b2 = P.fused ? w.conv_b[1] : nullptr;
  fa.mean[0] = a.chan_mean[0];
  fa.mean[1] = a.chan_mean[1];
  fa.mean[2] = a.chan_mean[2];
  fa.to_features = (P.fused && P.L == 2) ? 1 : 0;
  fa.out = fa.to_features ? ws + P.feat_off : ws + P.in_off[P.first_g];
  fa.K_feat = P.K;
  fa.out_rows = fa.to_features ? 0 : P.g[P.first_g].R;
  return fa;
}

static noscope_status launch_fc(const CnnPlan& P, const noscope_cnn_weights& w, uint8_t* ws,
                                const int64_t* n_dev, int64_t n_max, int64_t base, int64_t len,
                                float* logits, const int32_t* fq, const int32_t* pos_pf,
                                cudaStream_t st) {
  static DeviceOnce attr;
  if (attr.first())
    NS_CUDA_TRY(cudaFuncSetAttribute(fc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  FcArgs f{};
  f.feat = ws + P.feat_off;
  f.K = P.K;
  f.D = P.D;
  f.wpack = ws + P.fc_off;
  f.b1 = w.fc1_b;
  f.w2 = w.fc2_w;
  f.b2 = w.fc2_b;
  f.logits = logits;
  f.n_dev = n_dev;
  f.n_max = n_max;
  f.chunk_base = base;
  f.chunk_len = len;
  f.tmem_cols = tmem_cols_host(2 * P.D);
  f.ksplit = fc_ksplit(P.K);
  f.part = reinterpret_cast<float*>(ws + P.part_off);
  f.counters = reinterpret_cast<unsigned*>(ws + P.cnt_off);
  f.fq = fq;
  f.pos_pf = pos_pf;
  const size_t fsm = (size_t)kBStages * (128 * kFcKChunk * 2 + P.D * kFcKChunk * 2) +
                     (2 * kBStages + 1) * 8 + 32 + 1024;
  fc_kernel<<<(int)((len + 127) / 128) * f.ksplit, kCnnThreads, fsm, st>>>(f);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

noscope_status launch_cnn(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                          const uint8_t* small, int64_t small_pitch, const int32_t* idx,
                          const int64_t* n_dev, int64_t n_max, float* logits, void* ws_v,
                          uint32_t* status, cudaStream_t st) {
  (void)status;
  CnnPlan P;
  if (!make_plan(a, n_max, &P)) return NOSCOPE_INVALID_ARGUMENT;
  if (n_max <= 0) return NOSCOPE_OK;
  uint8_t* ws = reinterpret_cast<uint8_t*>(ws_v);
  noscope_status s = pack_weights(P, w, ws, st);   // canonical UMMA layouts
  if (s != NOSCOPE_OK) return s;
  if (fc_ksplit(P.K) > 1)   // FC split-K arrival counters start at zero (reset by their last CTA)
    NS_CUDA_TRY(cudaMemsetAsync(ws + P.cnt_off, 0, (size_t)(P.chunk / 128) * 4, st));
  for (int64_t base = 0; base < n_max; base += P.chunk) {
    const int64_t len = std::min<int64_t>(P.chunk, n_max - base);
    FusedArgs fa = fused_args(P, a, w, small, small_pitch, ws);
    fa.idx = idx;
    fa.n_dev = n_dev;
    fa.n_max = n_max;
    fa.chunk_base = base;
    fa.chunk_len = len;
    s = launch_conv12_fused(fa, (int)std::min<int64_t>(len, kNumSMs), st);
    if (s != NOSCOPE_OK) return s;
    for (int l = P.first_g; l < P.L; ++l) {
      ConvGArgs c{};
      c.g = P.g[l];
      c.in = ws + P.in_off[l];
      c.wpack = ws + P.gw_off[l];
      c.bias = w.conv_b[l];
      c.to_features = l == P.L - 1 ? 1 : 0;
      c.out = c.to_features ? ws + P.feat_off : ws + P.in_off[l + 1];
      c.out_rows = c.to_features ? 0 : P.g[l + 1].R;
      c.K_feat = P.K;
      c.n_dev = n_dev;
      c.n_max = n_max;
      c.chunk_base = base;
      c.chunk_len = len;
      s = c.g.tiled ? launch_convt(c, st) : launch_convg(c, st);
      if (s != NOSCOPE_OK) return s;
    }
    s = launch_fc(P, w, ws, n_dev, n_max, base, len, logits, nullptr, nullptr, st);
    if (s != NOSCOPE_OK) return s;
  }
  return NOSCOPE_OK;
}

// ----------------------------------------------------------- queue mode
bool cnn_queue_supported(const noscope_cnn_arch& a) {
  return cnn_arch_supported(a) && (a.base_filters == 32 || a.base_filters == 16) && a.n_conv == 2;
}

size_t cnn_queue_ws_bytes(const noscope_cnn_arch& a, int64_t n_max) {
  CnnPlan p;
  if (!cnn_queue_supported(a) || !make_plan(a, n_max, &p, true)) return 0;
  return p.total;
}

noscope_status cnn_queue_pack(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                              int64_t n_max, void* ws_v, cudaStream_t st) {
  CnnPlan P;
  if (!cnn_queue_supported(a) || !make_plan(a, n_max, &P, true)) return NOSCOPE_INVALID_ARGUMENT;
  uint8_t* ws = reinterpret_cast<uint8_t*>(ws_v);
  noscope_status s = pack_weights(P, w, ws, st);
  if (s != NOSCOPE_OK) return s;
  if (fc_ksplit(P.K) > 1)
    NS_CUDA_TRY(cudaMemsetAsync(ws + P.cnt_off, 0, (size_t)(P.chunk / 128) * 4, st));
  return NOSCOPE_OK;
}

noscope_status cnn_queue_conv(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                              const uint8_t* small, int64_t small_pitch, const FiredQueue& fq,
                              int qmode, int grid, int64_t n_max, void* ws_v, cudaStream_t st) {
  CnnPlan P;
  if (!cnn_queue_supported(a) || !make_plan(a, n_max, &P, true)) return NOSCOPE_INVALID_ARGUMENT;
  if (grid <= 0) return NOSCOPE_OK;
  uint8_t* ws = reinterpret_cast<uint8_t*>(ws_v);
  FusedArgs fa = fused_args(P, a, w, small, small_pitch, ws);
  fa.n_max = n_max;
  fa.chunk_len = P.chunk;
  fa.qmode = qmode;
  fa.fq = fq;
  return launch_conv12_fused(fa, grid, st);
}

noscope_status cnn_queue_fc(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                            const FiredQueue& fq, int64_t n_max, const int32_t* pos_pf,
                            float* logits, void* ws_v, cudaStream_t st) {
  CnnPlan P;
  if (!cnn_queue_supported(a) || !make_plan(a, n_max, &P, true)) return NOSCOPE_INVALID_ARGUMENT;
  if (n_max <= 0) return NOSCOPE_OK;
  return launch_fc(P, w, reinterpret_cast<uint8_t*>(ws_v),
                   reinterpret_cast<const int64_t*>(fq.count), n_max, 0, n_max, logits, fq.q,
                   pos_pf, st);
}

}  // namespace ns
