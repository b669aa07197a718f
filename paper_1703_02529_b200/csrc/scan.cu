// scan.cu — stream compaction ("batch input images"), routing
// and per-frame label resolution.
//
// Compaction is a single-pass decoupled look-back scan: tiles of 4096 items
// are claimed in launch order through an atomic counter, each tile publishes
// its aggregate then its inclusive prefix in one 64-bit word (flag | count),
// and successors accumulate predecessors' words walking backwards.  Output
// order is ascending (stable), so results are bit-identical to a serial scan.
//
// Label resolution follows the backward pointers of O8 without pointer
// chasing: among checked frames (tau = p * t_skip) a mode-1 suppression copies
// checked frame p - K, K = ceil(k / t_skip) (the checked frame that frame
// tau - k copies), so labels are a "last resolved value" scan inside each of
// the K residue classes; skipped frames copy their period's checked frame.
// Two launches: per-(class, segment) summaries, then apply with carries.
#include "common.cuh"
#include "internal.h"

namespace ns {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

NS_DEV unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
NS_DEV void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct ScanWs {
  unsigned long long* status;  // [ntiles]
  unsigned int* counter;       // tile ticket
};

size_t compact_ws_bytes(int64_t n) {
  int64_t tiles = (n + kScanTile - 1) / kScanTile + 1;
  return (size_t)(tiles * 8 + 64);
}
static ScanWs scan_ws_of(void* p, int64_t n) {
  ScanWs w;
  w.counter = reinterpret_cast<unsigned int*>(p);
  w.status = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(p) + 64);
  (void)n;
  return w;
}

// Block-wide exclusive scan of per-thread counts; *total = block sum.
NS_DEV uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;
  }
  __syncthreads();
  *total = warp_sums[nw - 1];
  uint32_t pre = warp == 0 ? 0u : warp_sums[warp - 1];
  return pre + x - v;
}

// Decoupled look-back: exclusive prefix of this tile (thread 0 does the walk).
NS_DEV uint64_t tile_lookback(ScanWs ws, int tile, uint32_t agg, uint64_t* s_excl) {
  if (threadIdx.x == 0) {
    uint64_t excl = 0;
    if (tile == 0) {
      st_relaxed(&ws.status[0], kFlagIncl | agg);
    } else {
      st_relaxed(&ws.status[tile], kFlagAgg | agg);
      int p = tile - 1;
      while (true) {
        unsigned long long v = ld_relaxed(&ws.status[p]);
        unsigned long long flag = v & ~kValMask;
        if (flag == 0) continue;
        excl += v & kValMask;
        if (flag == kFlagIncl) break;
        --p;
      }
      st_relaxed(&ws.status[tile], kFlagIncl | (excl + agg));
    }
    *s_excl = excl;
  }
  __syncthreads();
  return *s_excl;
}

NS_DEV int claim_tile(ScanWs ws, int* s_tile) {
  if (threadIdx.x == 0) *s_tile = (int)atomicAdd(ws.counter, 1u);
  __syncthreads();
  return *s_tile;
}

// ------------------------------------------------------------ fired frames
__global__ void __launch_bounds__(kScanThreads)
compact_fired_kernel(uint8_t* disp, double* score, int64_t n, int64_t tau0, int t_skip,
                     int32_t* idx_out, int64_t* count_out, ScanWs ws, int ntiles) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint64_t s_excl;
  __shared__ int s_tile;
  const int tile = claim_tile(ws, &s_tile);
  const int64_t base = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t flags = 0, cnt = 0;
#pragma unroll
  for (int e = 0; e < kScanItems; ++e) {
    const int64_t f = base + e;
    if (f < n) {
      const int64_t tau = tau0 + f;
      if (tau % t_skip != 0) {
        disp[f] = NOSCOPE_SKIPPED;
        if (score) score[f] = __longlong_as_double(0xFFF0000000000000ll);  // -inf
      } else if (disp[f] == NOSCOPE_FIRED) {
        flags |= 1u << e;
        ++cnt;
      }
    }
  }
  uint32_t total;
  uint32_t local = block_excl_scan(cnt, warp_sums, &total);
  uint64_t excl = tile_lookback(ws, tile, total, &s_excl);
  uint64_t pos = excl + local;
  if (idx_out) {
#pragma unroll
    for (int e = 0; e < kScanItems; ++e)
      if (flags & (1u << e)) idx_out[pos++] = (int32_t)(base + e);
  }
  if (count_out && tile == ntiles - 1 && threadIdx.x == 0) *count_out = (int64_t)(excl + total);
}

size_t compact_fired_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

noscope_status launch_compact_fired(const uint8_t* /*disp_in*/, uint8_t* disp, double* score,
                                    int64_t n, int64_t tau0, int t_skip, int32_t* idx_out,
                                    int64_t* count_out, void* scan_ws, cudaStream_t st) {
  const int ntiles = (int)compact_fired_tiles(n);
  if (ntiles == 0) {
    if (count_out) NS_CUDA_TRY(cudaMemsetAsync(count_out, 0, sizeof(int64_t), st));
    return NOSCOPE_OK;
  }
  NS_CUDA_TRY(cudaMemsetAsync(scan_ws, 0, compact_ws_bytes(n), st));
  compact_fired_kernel<<<ntiles, kScanThreads, 0, st>>>(disp, score, n, tau0, t_skip, idx_out,
                                                        count_out, scan_ws_of(scan_ws, n), ntiles);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

// ------------------------------------------------------------ routing
struct RouteArgs {
  float lo, hi;
  const float* logits;
  const int64_t* n_dev;
  int64_t n_max;
  const int32_t* frame_idx;  // nullable
  uint8_t* route_out;        // compact codes (nullable)
  uint8_t* route_pf;         // per-frame codes via frame_idx (nullable)
  int32_t* unc_out;
  int64_t* n_unc;
  int32_t* unc_pos_pf;       // per-frame position in the uncertain list (nullable)
  float* logits_pf;          // per-frame logits via frame_idx (nullable)
  unsigned long long* counters;  // [0] NEG, [1] POS (nullable)
  uint32_t* status;
};

__global__ void __launch_bounds__(kScanThreads)
route_kernel(RouteArgs A, ScanWs ws) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint64_t s_excl;
  __shared__ int s_tile;
  __shared__ unsigned int s_neg, s_pos;
  const int64_t n = A.n_dev ? min(*A.n_dev, A.n_max) : A.n_max;
  const int ntiles = (int)((n + kScanTile - 1) / kScanTile);
  const int tile = claim_tile(ws, &s_tile);
  if (n == 0) {
    if (tile == 0 && threadIdx.x == 0) *A.n_unc = 0;
    return;
  }
  if (tile >= ntiles) return;
  if (threadIdx.x == 0) s_neg = s_pos = 0;
  const int64_t base = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t flags = 0, cnt = 0, nneg = 0, npos = 0;
#pragma unroll
  for (int e = 0; e < kScanItems; ++e) {
    const int64_t i = base + e;
    if (i < n) {
      const float z = A.logits[i];
      uint8_t code;
      if (z < A.lo) {
        code = NOSCOPE_R_NEG;
        ++nneg;
      } else if (z > A.hi) {
        code = NOSCOPE_R_POS;
        ++npos;
      } else {
        code = NOSCOPE_R_UNC;
        flags |= 1u << e;
        ++cnt;
      }
      if (z != z) atomicOr(A.status, 2u);
      if (A.route_out) A.route_out[i] = code;
      if (A.frame_idx) {
        const int32_t f = A.frame_idx[i];
        if (A.route_pf) A.route_pf[f] = code;
        if (A.logits_pf) A.logits_pf[f] = z;
      }
    }
  }
  uint32_t total;
  uint32_t local = block_excl_scan(cnt, warp_sums, &total);
  if (A.counters) {
    if (nneg) atomicAdd(&s_neg, nneg);
    if (npos) atomicAdd(&s_pos, npos);
  }
  uint64_t excl = tile_lookback(ws, tile, total, &s_excl);
  uint64_t pos = excl + local;
#pragma unroll
  for (int e = 0; e < kScanItems; ++e)
    if (flags & (1u << e)) {
      const int64_t i = base + e;
      const int32_t f = A.frame_idx ? A.frame_idx[i] : (int32_t)i;
      if (A.unc_pos_pf) A.unc_pos_pf[f] = (int32_t)pos;
      A.unc_out[pos++] = f;
    }
  if (threadIdx.x == 0) {
    if (A.counters) {
      atomicAdd(&A.counters[0], (unsigned long long)s_neg);
      atomicAdd(&A.counters[1], (unsigned long long)s_pos);
    }
    if (tile == ntiles - 1) *A.n_unc = (int64_t)(excl + total);
  }
}

noscope_status launch_route(noscope_route r, const float* logits, const int64_t* n_dev,
                            int64_t n_max, const int32_t* frame_idx, uint8_t* route_out,
                            uint8_t* route_pf, int32_t* unc_out, int64_t* n_unc,
                            int32_t* unc_pos_pf, float* logits_pf, uint64_t* counters,
                            void* scan_ws, uint32_t* status, cudaStream_t st) {
  int ntiles = (int)((n_max + kScanTile - 1) / kScanTile);
  if (ntiles == 0) ntiles = 1;
  NS_CUDA_TRY(cudaMemsetAsync(scan_ws, 0, compact_ws_bytes(n_max), st));
  RouteArgs A{r.lo_logit, r.hi_logit, logits, n_dev, n_max, frame_idx, route_out, route_pf,
              unc_out, n_unc, unc_pos_pf, logits_pf,
              reinterpret_cast<unsigned long long*>(counters), status};
  route_kernel<<<ntiles, kScanThreads, 0, st>>>(A, scan_ws_of(scan_ws, n_max));
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

// ------------------------------------------------------------ labels
constexpr int kSeg = 32;
constexpr uint8_t kNone = 0xFF;

struct LabArgs {
  int64_t tau0, n;
  int mode, t_skip, K;
  int64_t p_first, nc;  // checked periods in chunk: p_first .. p_first + nc - 1
  int nseg;             // segments per class
  const uint8_t* disp;
  const uint8_t* route_pf;
  const int32_t* unc_pos_pf;
  const uint8_t* answers;
  const uint8_t* lab_hist;  // state label ring (slot tau % lh), nullable at unit start
  int lh;
  uint8_t* labels;
  uint8_t* route_out;  // nullable
  uint8_t* summary;    // [K][nseg]
};

// value of checked element e (frame f), or kNone if it copies its predecessor
NS_DEV uint8_t checked_value(const LabArgs& A, int64_t f) {
  const uint8_t d = A.disp[f];
  if (d == NOSCOPE_FIRED) {
    const uint8_t r = A.route_pf[f];
    if (r == NOSCOPE_R_NEG) return 0;
    if (r == NOSCOPE_R_POS) return 1;
    return A.answers[A.unc_pos_pf[f]] ? 1 : 0;
  }
  return A.mode == 0 ? 0 : kNone;  // suppressed
}
NS_DEV uint8_t hist_label(const LabArgs& A, int64_t tau) {
  return A.lab_hist ? A.lab_hist[tau % A.lh] : 0;
}

__global__ void labels_summary_kernel(LabArgs A) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)A.K * A.nseg) return;
  const int r = (int)(t / A.nseg), s = (int)(t % A.nseg);
  uint8_t last = kNone;
  for (int jj = 0; jj < kSeg; ++jj) {
    const int64_t e = (int64_t)(s * kSeg + jj) * A.K + r;
    if (e >= A.nc) break;
    const int64_t f = (A.p_first + e) * A.t_skip - A.tau0;
    const uint8_t v = checked_value(A, f);
    if (v != kNone) last = v;
  }
  A.summary[t] = last;
}

__global__ void labels_apply_kernel(LabArgs A) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {  // leading skipped frames copy the checked frame before the chunk
    const int64_t first_checked = A.p_first * A.t_skip;
    for (int64_t tau = A.tau0; tau < first_checked && tau < A.tau0 + A.n; ++tau) {
      const int64_t c = tau - tau % A.t_skip;
      A.labels[tau - A.tau0] = hist_label(A, c);
      if (A.route_out) A.route_out[tau - A.tau0] = NOSCOPE_R_SKIP;
    }
  }
  if (t >= (int64_t)A.K * A.nseg) return;
  const int r = (int)(t / A.nseg), s = (int)(t % A.nseg);
  uint8_t carry = kNone;
  if (A.mode == 1) {
    for (int ss = s - 1; ss >= 0 && carry == kNone; --ss) carry = A.summary[(int64_t)r * A.nseg + ss];
    if (carry == kNone) {
      const int64_t p_pred = A.p_first + r - A.K;  // predecessor of the class head
      carry = p_pred >= 0 ? hist_label(A, p_pred * A.t_skip) : 0;
    }
  }
  for (int jj = 0; jj < kSeg; ++jj) {
    const int64_t e = (int64_t)(s * kSeg + jj) * A.K + r;
    if (e >= A.nc) break;
    const int64_t tau = (A.p_first + e) * A.t_skip;
    const int64_t f = tau - A.tau0;
    uint8_t v = checked_value(A, f);
    const uint8_t d = A.disp[f];
    if (v == kNone) v = carry;
    carry = v;
    A.labels[f] = v;
    if (A.route_out)
      A.route_out[f] = d == NOSCOPE_FIRED ? A.route_pf[f] : (uint8_t)NOSCOPE_R_SUPP;
    for (int q = 1; q < A.t_skip && f + q < A.n; ++q) {
      A.labels[f + q] = v;
      if (A.route_out) A.route_out[f + q] = NOSCOPE_R_SKIP;
    }
  }
}

size_t labels_ws_bytes(int64_t n) { return (size_t)(n / kSeg + 4096); }

noscope_status launch_labels(const noscope_dd_config& cfg, int64_t tau0, int64_t n,
                             const uint8_t* disp, const uint8_t* route_pf,
                             const int32_t* unc_pos_pf, const uint8_t* answers,
                             const uint8_t* lab_hist, uint8_t* labels, uint8_t* route_out,
                             void* lws, cudaStream_t st) {
  LabArgs A{};
  A.tau0 = tau0;
  A.n = n;
  A.mode = cfg.mode;
  A.t_skip = cfg.t_skip_frames;
  A.K = cfg.mode == 1 ? (cfg.t_diff_frames + A.t_skip - 1) / A.t_skip : 1;
  A.p_first = (tau0 + A.t_skip - 1) / A.t_skip;
  const int64_t p_end = (tau0 + n + A.t_skip - 1) / A.t_skip;
  A.nc = p_end - A.p_first;
  if (A.nc < 0) A.nc = 0;
  const int64_t per_class = (A.nc + A.K - 1) / A.K;
  A.nseg = (int)((per_class + kSeg - 1) / kSeg);
  A.disp = disp;
  A.route_pf = route_pf;
  A.unc_pos_pf = unc_pos_pf;
  A.answers = answers;
  A.lab_hist = lab_hist;
  A.lh = state_label_len(cfg);
  A.labels = labels;
  A.route_out = route_out;
  A.summary = reinterpret_cast<uint8_t*>(lws);
  const int64_t threads = (int64_t)A.K * A.nseg;
  const int blocks = (int)std::max<int64_t>(1, (threads + 255) / 256);
  if (cfg.mode == 1 && threads > 0) {
    labels_summary_kernel<<<blocks, 256, 0, st>>>(A);
    NS_LAUNCH_CHECK();
    count_launch();
  }
  labels_apply_kernel<<<blocks, 256, 0, st>>>(A);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

}  // namespace ns
