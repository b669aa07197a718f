// dd.cu — frame downsampling + difference detector (§5).
//
// dd_downsample_kernel: persistent, 2 CTAs/SM.  Each CTA walks its share of the
//   frames that must be downsampled (checked frames, plus mode-1 anchors), one
//   output row ("band") at a time.  A band = the source rows
//   [floor(iH/h), floor((i+1)H/h)) = one contiguous byte range of the frame,
//   fetched by a single cp.async.bulk (TMA 1-D) into a 4-stage shared-memory
//   ring with mbarrier completion, evict-first L2 policy (each source byte is
//   read exactly once).  Compute per band: (1) vertical sums of every source
//   byte column with SWAR 2x16-bit lanes, (2) horizontal box sums -> the
//   rounded integer mean G (O1, reading R-1) -> small frame row stored to HBM
//   (the CNN's input) and, in mode 0, the exact integer SSD against the
//   reference image (kept in smem) accumulated per thread / per LR block.
//   At frame end the fp64 score and the disposition are written (O3/O4).
// dd_lag_score_kernel: mode 1 (anchor = frame tau-k) scores, one CTA per
//   checked frame, reading both small frames (L2-resident) — the anchor may be
//   produced by another CTA, so this runs after the downsample pass.
// dd_state_update_kernel: carries the last k small frames / labels of a chunk
//   into the caller's stream state.
#include "common.cuh"
#include "internal.h"

namespace ns {

uint64_t& launch_counter() {
  static thread_local uint64_t c = 0;
  return c;
}

constexpr int kDsThreads = 256;
constexpr int kDsStages = 4;

struct DsArgs {
  const uint8_t* frames;
  int64_t frame_pitch;
  int W, H, RB;  // RB = W*3 bytes per source row
  int out_w, out_h;
  uint8_t* small;
  int64_t small_pitch;
  NeededSet need;
  int mode, metric, grid;
  const uint8_t* ref;
  const float* lr_w;
  float lr_b;
  double delta;
  double* score;
  uint8_t* disp;
  uint32_t* status;
  int stage_bytes;
  int fast;  // RB % 16 == 0 : SWAR vector path
};

// --------------------------------------------------------------- scoring
// Per-thread SSD accumulation; thread owns output column (j, c).
struct SsdAcc {
  uint64_t total;   // global metric
  uint32_t blk;     // blocked metric: current block row partial
  int cur_bi;
};

NS_DEV int block_of(int i, int n, int g) {
  int step = n / g;
  int b = i / step;
  return b < g - 1 ? b : g - 1;
}

NS_DEV void ssd_add(SsdAcc& a, uint32_t d2, int i, int j, const DsGeom& geo,
                    unsigned long long* blk_ssd) {
  if (geo.metric == 0) {
    a.total += d2;
  } else {
    int bi = block_of(i, geo.out_h, geo.grid);
    if (bi != a.cur_bi) {
      if (a.cur_bi >= 0 && a.blk)
        atomicAdd(&blk_ssd[a.cur_bi * geo.grid + block_of(j, geo.out_w, geo.grid)],
                  (unsigned long long)a.blk);
      a.cur_bi = bi;
      a.blk = 0;
    }
    a.blk += d2;
  }
}

// Finish a frame's score: block-wide reduction, fp64 score (O3), disposition (O4).
// Must be called by all threads of the CTA.  `red` = 32 u64 scratch.
NS_DEV void ssd_finish(SsdAcc& a, int j_thread, bool active, const DsGeom& geo,
                       unsigned long long* blk_ssd, unsigned long long* red, double* score_slot,
                       uint8_t* disp_slot, uint32_t* status) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (geo.metric == 0) {
    unsigned long long v = active ? a.total : 0ull;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      double sc = (double)s / (double)(geo.out_w * geo.out_h * 3);
      *score_slot = sc;
      *disp_slot = sc > geo.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
    }
  } else {
    if (active && a.cur_bi >= 0 && a.blk)
      atomicAdd(&blk_ssd[a.cur_bi * geo.grid + block_of(j_thread, geo.out_w, geo.grid)],
                (unsigned long long)a.blk);
    __syncthreads();
    if (tid == 0) {
      const int g = geo.grid;
      const int sh = geo.out_h / g, sw = geo.out_w / g;
      double z = (double)geo.lr_b;
      for (int bi = 0; bi < g; ++bi) {
        int rows = (bi < g - 1) ? sh : geo.out_h - (g - 1) * sh;
        for (int bj = 0; bj < g; ++bj) {
          int cols = (bj < g - 1) ? sw : geo.out_w - (g - 1) * sw;
          double m = (double)blk_ssd[bi * g + bj] / (double)(rows * cols * 3);
          z = __dadd_rn(z, __dmul_rn((double)geo.lr_w[bi * g + bj], m));
        }
      }
      if (z != z) atomicOr(status, 1u);
      *score_slot = z;
      *disp_slot = z > geo.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
    }
    __syncthreads();
    for (int t = tid; t < geo.grid * geo.grid; t += blockDim.x) blk_ssd[t] = 0ull;
  }
  a.total = 0;
  a.blk = 0;
  a.cur_bi = -1;
  __syncthreads();
}

// ------------------------------------------------------ downsample kernel
__global__ void __launch_bounds__(kDsThreads, 2)
dd_downsample_kernel(DsArgs A, DsGeom geo) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;                                        // S * stage_bytes
  uint16_t* colsum = reinterpret_cast<uint16_t*>(smem + kDsStages * A.stage_bytes);  // 2 * RB
  uint8_t* ref_s = reinterpret_cast<uint8_t*>(colsum + 2 * ((A.RB + 7) & ~7));
  const int small_bytes = A.out_w * A.out_h * 3;
  unsigned long long* blk_ssd =
      reinterpret_cast<unsigned long long*>(ref_s + ((small_bytes + 15) & ~15));
  unsigned long long* red = blk_ssd + ((geo.grid * geo.grid + 1) & ~1);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 32);

  const int tid = threadIdx.x;
  const int64_t m_count = A.need.m1 - A.need.m0;
  const int64_t my_frames =
      m_count > blockIdx.x ? (m_count - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total_seq = my_frames * A.out_h;
  const bool score_here = (A.mode == 0);

  if (tid == 0) {
    for (int s = 0; s < kDsStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  if (score_here) {
    for (int t = tid; t < small_bytes; t += blockDim.x) ref_s[t] = A.ref[t];
    for (int t = tid; t < geo.grid * geo.grid; t += blockDim.x) blk_ssd[t] = 0ull;
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  // seq -> (frame, band) and its byte range
  auto issue = [&](int64_t seq) {
    int64_t ml = seq / A.out_h;
    int i = (int)(seq - ml * A.out_h);
    int64_t m = A.need.m0 + blockIdx.x + ml * gridDim.x;
    int64_t f = A.need.frame_of(m);
    int r0 = (i * A.H) / A.out_h, r1 = ((i + 1) * A.H) / A.out_h;
    int64_t b0 = (int64_t)r0 * A.RB, b1 = (int64_t)r1 * A.RB;
    int64_t a0 = b0 & ~(int64_t)15, a1 = (b1 + 15) & ~(int64_t)15;
    int s = (int)(seq % kDsStages);
    mbar_arrive_expect_tx(&full[s], (uint32_t)(a1 - a0));
    bulk_g2s_evict_first(stages + (size_t)s * A.stage_bytes, A.frames + f * A.frame_pitch + a0,
                         (uint32_t)(a1 - a0), &full[s], pol);
  };
  if (tid == 0)
    for (int64_t q = 0; q < kDsStages - 1 && q < total_seq; ++q) issue(q);

  const int n_out = A.out_w * 3;
  SsdAcc acc{0, 0, -1};

  for (int64_t seq = 0; seq < total_seq; ++seq) {
    const int64_t ml = seq / A.out_h;
    const int i = (int)(seq - ml * A.out_h);
    const int64_t m = A.need.m0 + blockIdx.x + ml * gridDim.x;
    const int64_t f = A.need.frame_of(m);
    const int s = (int)(seq % kDsStages);
    if (tid == 0 && seq + kDsStages - 1 < total_seq) issue(seq + kDsStages - 1);
    mbar_wait(&full[s], (uint32_t)((seq / kDsStages) & 1));

    const int r0 = (i * A.H) / A.out_h, r1 = ((i + 1) * A.H) / A.out_h;
    const int nrows = r1 - r0;
    const int off = (int)(((int64_t)r0 * A.RB) & 15);
    const uint8_t* band = stages + (size_t)s * A.stage_bytes + off;
    uint16_t* cs = colsum + (seq & 1) * ((A.RB + 7) & ~7);

    // (1) vertical sums: SWAR, two 16-bit lanes per 32-bit word
    if (A.fast) {
      const int nvec = A.RB >> 3;  // 8-byte units
      for (int v = tid; v < nvec; v += blockDim.x) {
        uint32_t lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
        const uint2* p = reinterpret_cast<const uint2*>(band) + v;
        for (int r = 0; r < nrows; ++r) {
          uint2 w = p[(size_t)r * (A.RB >> 3)];
          lo0 += w.x & 0x00FF00FFu;
          hi0 += (w.x >> 8) & 0x00FF00FFu;
          lo1 += w.y & 0x00FF00FFu;
          hi1 += (w.y >> 8) & 0x00FF00FFu;
        }
        uint4 o;
        o.x = (lo0 & 0xFFFFu) | (hi0 << 16);          // bytes 0,1
        o.y = (lo0 >> 16) | (hi0 & 0xFFFF0000u);      // bytes 2,3
        o.z = (lo1 & 0xFFFFu) | (hi1 << 16);
        o.w = (lo1 >> 16) | (hi1 & 0xFFFF0000u);
        reinterpret_cast<uint4*>(cs)[v] = o;
      }
    } else {
      for (int b = tid; b < A.RB; b += blockDim.x) {
        uint32_t sum = 0;
        for (int r = 0; r < nrows; ++r) sum += band[(size_t)r * A.RB + b];
        cs[b] = (uint16_t)sum;
      }
    }
    __syncthreads();

    // (2) horizontal box sums -> G, store, SSD vs reference image
    uint8_t* dst = A.small + f * A.small_pitch + (size_t)i * n_out;
    for (int t = tid; t < n_out; t += blockDim.x) {
      const int j = t / 3, c = t - 3 * (t / 3);
      const int q0 = (j * A.W) / A.out_w, q1 = ((j + 1) * A.W) / A.out_w;
      uint32_t S = 0;
      for (int q = q0; q < q1; ++q) S += cs[q * 3 + c];
      const uint32_t n = (uint32_t)nrows * (uint32_t)(q1 - q0);
      const uint32_t G = (2u * S + n) / (2u * n);
      dst[t] = (uint8_t)G;
      if (score_here) {
        int d = (int)G - (int)ref_s[i * n_out + t];
        ssd_add(acc, (uint32_t)(d * d), i, j, geo, blk_ssd);
      }
    }

    if (i == A.out_h - 1 && score_here) {
      // frame complete: only checked frames are scored (in mode 0 every
      // downsampled frame is checked)
      __syncthreads();
      ssd_finish(acc, tid / 3, tid < n_out, geo, blk_ssd, red, &A.score[f], &A.disp[f], A.status);
    }
  }
}

// ------------------------------------------------------ mode 1 lag scores
struct LagArgs {
  const uint8_t* small;
  int64_t small_pitch;
  const uint8_t* ring;  // state ring: k slots of small_bytes (slot pitch ring_pitch)
  int64_t ring_pitch;
  int64_t tau0, n;
  int k, t_skip, out_w, out_h;
  int64_t p0, p1;  // checked periods: tau = p * t_skip in [tau0, tau0+n)
  double* score;
  uint8_t* disp;
  uint32_t* status;
};

__global__ void __launch_bounds__(kDsThreads)
dd_lag_score_kernel(LagArgs A, DsGeom geo) {
  __shared__ unsigned long long blk_ssd[kMaxGrid * kMaxGrid];
  __shared__ unsigned long long red[32];
  const int tid = threadIdx.x;
  const int n_out = A.out_w * 3;
  for (int t = tid; t < geo.grid * geo.grid; t += blockDim.x) blk_ssd[t] = 0ull;
  __syncthreads();
  for (int64_t p = A.p0 + blockIdx.x; p < A.p1; p += gridDim.x) {
    const int64_t tau = p * A.t_skip;
    const int64_t f = tau - A.tau0;
    if (tau < A.k) {  // forced fire: no anchor yet (reading R-8)
      if (tid == 0) {
        A.score[f] = __longlong_as_double(0x7FF0000000000000ll);
        A.disp[f] = NOSCOPE_FIRED;
      }
      continue;
    }
    const int64_t fa = f - A.k;
    const uint8_t* G = A.small + f * A.small_pitch;
    const uint8_t* Aimg = fa >= 0 ? A.small + fa * A.small_pitch
                                  : A.ring + ((tau - A.k) % A.k) * A.ring_pitch;
    SsdAcc acc{0, 0, -1};
    if (tid < n_out) {
      const int j = tid / 3;
      for (int i = 0; i < A.out_h; ++i) {
        int d = (int)G[i * n_out + tid] - (int)Aimg[i * n_out + tid];
        ssd_add(acc, (uint32_t)(d * d), i, j, geo, blk_ssd);
      }
    }
    ssd_finish(acc, tid / 3, tid < n_out, geo, blk_ssd, red, &A.score[f], &A.disp[f], A.status);
  }
}

// ------------------------------------------------------ state update
__global__ void dd_state_update_kernel(const uint8_t* small, int64_t small_pitch, uint8_t* ring,
                                       int64_t ring_pitch, int k, int small_bytes, int64_t tau0,
                                       int64_t n, const uint8_t* labels, uint8_t* lab_hist,
                                       int lh) {
  // frames tau in [tau0 + n - k, tau0 + n) -> ring slot tau % k
  const int64_t first = n - k > 0 ? n - k : 0;
  for (int64_t f = first + blockIdx.x; f < n && ring; f += gridDim.x) {
    const int64_t tau = tau0 + f;
    const uint8_t* src = small + f * small_pitch;
    uint8_t* dst = ring + (tau % k) * ring_pitch;
    for (int t = threadIdx.x; t < small_bytes; t += blockDim.x) dst[t] = src[t];
  }
  if (labels && blockIdx.x == 0) {
    const int64_t lf = n - lh > 0 ? n - lh : 0;
    for (int64_t f = lf + threadIdx.x; f < n; f += blockDim.x)
      lab_hist[(tau0 + f) % lh] = labels[f];
  }
}

// ===================================================================== host
size_t ds_smem_bytes(int W, int H, int out_w, int out_h, int grid, int* stage_bytes_out) {
  const int RB = W * 3;
  int max_rows = 0;
  int stage = 0;
  for (int i = 0; i < out_h; ++i) {
    int r0 = (i * H) / out_h, r1 = ((i + 1) * H) / out_h;
    int64_t b0 = (int64_t)r0 * RB, b1 = (int64_t)r1 * RB;
    int64_t a0 = b0 & ~15ll, a1 = (b1 + 15) & ~15ll;
    if ((int)(a1 - a0) > stage) stage = (int)(a1 - a0);
    if (r1 - r0 > max_rows) max_rows = r1 - r0;
  }
  stage = (stage + 127) & ~127;
  if (stage_bytes_out) *stage_bytes_out = stage;
  const int small_bytes = out_w * out_h * 3;
  size_t b = (size_t)kDsStages * stage;
  b += 2 * (size_t)((RB + 7) & ~7) * sizeof(uint16_t);
  b += (size_t)((small_bytes + 15) & ~15);
  b += (size_t)(((grid * grid + 1) & ~1) + 32) * 8;
  b += kDsStages * 8;
  return b;
}

noscope_status launch_diff_detect(const noscope_dd_config& cfg, const uint8_t* frames,
                                  const noscope_frames_desc& desc, int64_t n, int64_t tau0,
                                  uint8_t* state, uint8_t* small, int64_t small_pitch,
                                  double* score, uint8_t* disp, uint32_t* status,
                                  cudaStream_t st, Prof* prof) {
  DsGeom geo{};
  geo.out_w = cfg.out_w;
  geo.out_h = cfg.out_h;
  geo.metric = cfg.metric;
  geo.grid = cfg.metric == 1 ? cfg.grid : 1;
  geo.lr_w = cfg.lr_weights;
  geo.lr_b = cfg.lr_bias;
  geo.delta = cfg.delta_diff;
  const int k = cfg.mode == 1 ? cfg.t_diff_frames : 0;

  NeededSet need = make_needed_set(cfg, tau0, n);
  if (need.m1 > need.m0) {
    DsArgs A{};
    A.frames = frames;
    A.frame_pitch = desc.frame_pitch;
    A.W = desc.width;
    A.H = desc.height;
    A.RB = desc.width * 3;
    A.out_w = cfg.out_w;
    A.out_h = cfg.out_h;
    A.small = small;
    A.small_pitch = small_pitch;
    A.need = need;
    A.mode = cfg.mode;
    A.metric = cfg.metric;
    A.grid = geo.grid;
    A.ref = cfg.ref_image;
    A.lr_w = cfg.lr_weights;
    A.lr_b = cfg.lr_bias;
    A.delta = cfg.delta_diff;
    A.score = score;
    A.disp = disp;
    A.status = status;
    A.fast = (A.RB % 16) == 0;
    size_t smem = ds_smem_bytes(desc.width, desc.height, cfg.out_w, cfg.out_h, geo.grid,
                                &A.stage_bytes);
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(dd_downsample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024);
      attr_set = true;
    }
    int64_t frames_needed = need.m1 - need.m0;
    int grid = (int)std::min<int64_t>(frames_needed, 2 * kNumSMs);
    dd_downsample_kernel<<<grid, kDsThreads, smem, st>>>(A, geo);
    NS_LAUNCH_CHECK();
    count_launch();
  }
  prof_mark(prof, st);
  if (cfg.mode == 1) {
    LagArgs L{};
    L.small = small;
    L.small_pitch = small_pitch;
    L.ring = state;
    L.ring_pitch = state_ring_pitch(cfg);
    L.tau0 = tau0;
    L.n = n;
    L.k = k;
    L.t_skip = cfg.t_skip_frames;
    L.out_w = cfg.out_w;
    L.out_h = cfg.out_h;
    L.p0 = (tau0 + cfg.t_skip_frames - 1) / cfg.t_skip_frames;
    L.p1 = (tau0 + n + cfg.t_skip_frames - 1) / cfg.t_skip_frames;
    L.score = score;
    L.disp = disp;
    L.status = status;
    if (L.p1 > L.p0) {
      int grid = (int)std::min<int64_t>(L.p1 - L.p0, 16 * kNumSMs);
      dd_lag_score_kernel<<<grid, kDsThreads, 0, st>>>(L, geo);
      NS_LAUNCH_CHECK();
      count_launch();
    }
  }
  return NOSCOPE_OK;
}

noscope_status launch_state_update(const noscope_dd_config& cfg, const uint8_t* small,
                                   int64_t small_pitch, uint8_t* state, int64_t tau0, int64_t n,
                                   const uint8_t* labels, cudaStream_t st) {
  if (!state || n <= 0) return NOSCOPE_OK;
  uint8_t* ring = cfg.mode == 1 ? state : nullptr;
  const int k = cfg.mode == 1 ? cfg.t_diff_frames : 1;
  uint8_t* lab = state + state_ring_bytes(cfg);
  const int lh = state_label_len(cfg);
  int grid = ring ? (int)std::min<int64_t>(std::min<int64_t>(n, k), 256) : 1;
  dd_state_update_kernel<<<grid, 256, 0, st>>>(small, small_pitch, ring, state_ring_pitch(cfg), k,
                                               cfg.out_w * cfg.out_h * 3, tau0, n, labels, lab,
                                               lh);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

}  // namespace ns
