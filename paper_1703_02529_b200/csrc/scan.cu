// scan.cu — stream compaction ("batch input images"), routing
// and per-frame label resolution.
//
// Compaction of the FIRED frames is one persistent two-phase launch (count per
// contiguous range, grid barrier, write) — see compact_fired_kernel.  Routing's
// compaction of the uncertain frames is a single-pass decoupled look-back scan:
// tiles of 8192 items are claimed in launch order through an atomic counter,
// each tile publishes its aggregate then its inclusive prefix in one 64-bit word
// (flag | count), and successors accumulate predecessors' words walking
// backwards.  Both outputs are ascending (stable), bit-identical to a serial scan.
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

constexpr int kScanThreads = 512;
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

// Decoupled look-back: exclusive prefix of this tile.  Warp 0 inspects the 32
// preceding tiles' status words at once: if one of them holds an inclusive prefix,
// the nearest such tile ends the walk (sum of the words up to it); otherwise all 32
// aggregates are added and the window moves 32 tiles back.
NS_DEV uint64_t tile_lookback(ScanWs ws, int tile, uint32_t agg, uint64_t* s_excl) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed(&ws.status[0], kFlagIncl | agg);
    } else {
      if (lane == 0) st_relaxed(&ws.status[tile], kFlagAgg | agg);
      int p = tile - 1;  // window [p - 31, p]; lane l reads tile p - l
      while (true) {
        const int q = p - lane;
        unsigned long long v = q >= 0 ? ld_relaxed(&ws.status[q]) : kFlagIncl;
        while (__any_sync(0xffffffffu, (v & ~kValMask) == 0)) {
          if ((v & ~kValMask) == 0) v = ld_relaxed(&ws.status[q]);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, (v & ~kValMask) == kFlagIncl);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive tile (or the window)
        uint64_t x = lane <= stop ? (v & kValMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        excl += x;
        if (incl) break;
        p -= 32;
      }
      if (lane == 0) st_relaxed(&ws.status[tile], kFlagIncl | (excl + agg));
    }
    if (lane == 0) *s_excl = excl;
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
// Tile-local stable write-out: the tile's selected indices are staged in smem in
// scan order, then stored as one coalesced run at the tile's global offset.
NS_DEV void store_run(int32_t* out, uint64_t excl, uint32_t total, const int32_t* idx_s) {
  for (uint32_t k = threadIdx.x; k < total; k += blockDim.x) out[excl + k] = idx_s[k];
}

// Compaction of the FIRED frames (O5) as one persistent launch in two phases,
// all G CTAs co-resident, CTA c owning the contiguous tile range
// [c*T/G, (c+1)*T/G) of 8,192-frame tiles:
//   phase 1: stream the range, count FIRED frames (and apply the t_skip rewrite:
//            SKIPPED + score -inf in global memory); publish the range count;
//   grid barrier (atomic arrival counter, acquire spin);
//   phase 2: offset = sum of the lower ranges' counts; stream the range again and
//            write the ascending indices, tile by tile (block scan, indices staged
//            in smem, one coalesced run per tile).
// Both phases prefetch kCStages tiles ahead with cp.async.bulk into a smem ring
// (one mbarrier per stage), so every pass streams at HBM rate; there is no
// look-back chain (a single-pass decoupled look-back is bound by one L2 round trip
// per round of G tiles).  At the cascade's chunk sizes phase 2 re-reads from L2.
// Tail or misaligned tiles are read directly from global memory.
constexpr int kCThreads = 256, kCItems = 32, kCTile = kCThreads * kCItems, kCStages = 4;
static_assert(NOSCOPE_FIRED == 2, "SWAR compare below tests bytes == 0x02");

NS_DEV unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kCThreads)
compact_fired_kernel(uint8_t* disp, double* score, int64_t n, int64_t tau0, int t_skip,
                     int32_t* idx_out, int64_t* count_out, ScanWs ws, int ntiles, int vec) {
  extern __shared__ __align__(128) uint8_t csm[];
  uint8_t* ring = csm;                                            // kCStages x kCTile
  uint64_t* full = reinterpret_cast<uint64_t*>(csm + kCStages * kCTile);
  uint32_t* warp_sums = reinterpret_cast<uint32_t*>(full + kCStages);  // [32]
  uint64_t* s_off = reinterpret_cast<uint64_t*>(warp_sums + 32);
  int32_t* idx_s = reinterpret_cast<int32_t*>(s_off + 2);         // kCTile staged indices
  const int tid = threadIdx.x, G = gridDim.x, c = blockIdx.x;
  const int t0 = (int)(((int64_t)ntiles * c) / G), t1 = (int)(((int64_t)ntiles * (c + 1)) / G);
  const int nt = t1 - t0;
  auto bulk_ok = [&](int t) { return vec && (int64_t)(t + 1) * kCTile <= n; };
  // k-th fill of the ring (k counts over both passes): tile t0 + k % nt into stage k % kCStages
  auto fill = [&](int k) {
    const int st = k % kCStages;
    const int t = t0 + (k < nt ? k : k - nt);
    if (k < 2 * nt && bulk_ok(t)) {
      mbar_arrive_expect_tx(&full[st], (uint32_t)kCTile);
      bulk_g2s(ring + (size_t)st * kCTile, disp + (int64_t)t * kCTile, (uint32_t)kCTile, &full[st]);
    } else {
      mbar_arrive(&full[st]);  // keeps the stage's phase count in step
    }
  };
  if (tid == 0) {
    for (int st = 0; st < kCStages; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
    for (int k = 0; k < kCStages; ++k) fill(k);
  }
  __syncthreads();
  // this thread's 16 frames of the k-th tile of the range: FIRED flags after the t_skip rule
  auto load_flags = [&](int k, bool rewrite) -> uint32_t {
    const int st = k % kCStages;
    mbar_wait(&full[st], (uint32_t)((k / kCStages) & 1));
    const int t = t0 + (k < nt ? k : k - nt);
    const int64_t base = (int64_t)t * kCTile + (int64_t)tid * kCItems;
    uint8_t d[kCItems];
    if (bulk_ok(t)) {
      const uint4* vp = reinterpret_cast<const uint4*>(ring + (size_t)st * kCTile + tid * kCItems);
      const uint4 v0 = vp[0], v1 = vp[1];
      const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      if (t_skip == 1) {  // SWAR: FIRED bytes -> 4-bit masks (byte e -> bit e)
        uint32_t flags = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          flags |= (((__vcmpeq4(w[j], 0x02020202u) & 0x01010101u) * 0x01020408u) >> 24) << (4 * j);
        return flags;
      }
#pragma unroll
      for (int e = 0; e < kCItems; ++e) d[e] = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
    } else {
#pragma unroll
      for (int e = 0; e < kCItems; ++e) d[e] = base + e < n ? disp[base + e] : (uint8_t)0;
    }
    uint32_t flags = 0;
    if (t_skip == 1) {
#pragma unroll
      for (int e = 0; e < kCItems; ++e)
        if (d[e] == NOSCOPE_FIRED && base + e < n) flags |= 1u << e;
    } else {
      int r = (int)((tau0 + base) % t_skip);  // tau mod t_skip, advanced incrementally
#pragma unroll
      for (int e = 0; e < kCItems; ++e) {
        const int64_t f = base + e;
        if (f < n) {
          if (r != 0) {
            if (rewrite) {
              disp[f] = NOSCOPE_SKIPPED;
              if (score) score[f] = __longlong_as_double(0xFFF0000000000000ll);  // -inf
            }
          } else if (d[e] == NOSCOPE_FIRED) {
            flags |= 1u << e;
          }
        }
        if (++r == t_skip) r = 0;
      }
    }
    return flags;
  };

  // ---- phase 1: count
  uint32_t mine = 0;
  for (int k = 0; k < nt; ++k) {
    mine += __popc(load_flags(k, true));
    __syncthreads();                    // every thread is done with stage k % kCStages
    if (tid == 0) fill(k + kCStages);
  }
  uint32_t range_total;
  block_excl_scan(mine, warp_sums, &range_total);
  if (tid == 0) {
    st_relaxed(&ws.status[c], (unsigned long long)range_total);
    __threadfence();
    atomicAdd(ws.counter, 1u);
    while (ld_acquire_gpu(ws.counter) < (unsigned)G) {
    }
    uint64_t off = 0;
    for (int q = 0; q < c; ++q) off += ld_relaxed(&ws.status[q]);
    *s_off = off;
    if (c == G - 1 && count_out) *count_out = (int64_t)(off + range_total);
  }
  __syncthreads();
  uint64_t off = *s_off;

  // ---- phase 2: write the ascending indices
  for (int k = nt; k < 2 * nt; ++k) {
    const uint32_t flags = load_flags(k, false);
    uint32_t total;
    const uint32_t local = block_excl_scan((uint32_t)__popc(flags), warp_sums, &total);
    if (tid == 0) fill(k + kCStages);   // block_excl_scan synced: stage free
    const int64_t base = (int64_t)(t0 + k - nt) * kCTile + (int64_t)tid * kCItems;
    uint32_t q = local;
    for (uint32_t f = flags; f; f &= f - 1) idx_s[q++] = (int32_t)(base + __ffs(f) - 1);
    __syncthreads();
    if (idx_out) store_run(idx_out, off, total, idx_s);
    off += total;
    __syncthreads();                    // idx_s / warp_sums reuse
  }
}

static size_t compact_smem_bytes() {
  return (size_t)kCStages * kCTile + kCStages * 8 + 32 * 4 + 16 + (size_t)kCTile * 4;
}

size_t compact_fired_tiles(int64_t n) { return (n + kCTile - 1) / kCTile; }

noscope_status launch_compact_fired(const uint8_t* /*disp_in*/, uint8_t* disp, double* score,
                                    int64_t n, int64_t tau0, int t_skip, int32_t* idx_out,
                                    int64_t* count_out, void* scan_ws, cudaStream_t st) {
  const int ntiles = (int)compact_fired_tiles(n);
  if (ntiles == 0) {
    if (count_out) NS_CUDA_TRY(cudaMemsetAsync(count_out, 0, sizeof(int64_t), st));
    return NOSCOPE_OK;
  }
  NS_CUDA_TRY(cudaMemsetAsync(scan_ws, 0, compact_ws_bytes(n), st));
  const int vec = (reinterpret_cast<uintptr_t>(disp) & 15) == 0;
  const size_t smem = compact_smem_bytes();
  static DeviceInt occ;
  int per_sm = occ.get();
  if (per_sm == 0) {
    NS_CUDA_TRY(cudaFuncSetAttribute(compact_fired_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compact_fired_kernel, kCThreads, smem));
    if (per_sm < 1) per_sm = 1;
    occ.set(per_sm);
  }
  int sms = kNumSMs, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // persistent and co-resident (look-back waits only on earlier-claimed tiles)
  const int grid = std::min(ntiles, per_sm * sms);
  NS_CUDA_TRY(launch_cooperative(compact_fired_kernel, grid, kCThreads, smem, st, disp, score, n, tau0, t_skip,
                                 idx_out, count_out, scan_ws_of(scan_ws, n), ntiles, vec));
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
  int vec;                   // logits and route_out 16-byte aligned
};

__global__ void __launch_bounds__(kScanThreads)
route_kernel(RouteArgs A, ScanWs ws) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint64_t s_excl;
  __shared__ int s_tile;
  __shared__ unsigned int s_neg, s_pos;
  __shared__ int32_t idx_s[kScanTile];
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
  const bool full = A.vec && base + kScanItems <= n;
  float zv[kScanItems];
  if (full) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      const float4 v = reinterpret_cast<const float4*>(A.logits + base)[q];
      zv[4 * q] = v.x; zv[4 * q + 1] = v.y; zv[4 * q + 2] = v.z; zv[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < kScanItems; ++e) zv[e] = base + e < n ? A.logits[base + e] : 0.f;
  }
  uint32_t flags = 0, cnt = 0, nneg = 0, npos = 0, nan = 0;
  uint8_t code[kScanItems];
#pragma unroll
  for (int e = 0; e < kScanItems; ++e) {
    const float z = zv[e];
    const bool in = base + e < n;
    // NEG iff z < lo, POS iff z > hi, else UNCERTAIN (R-5; NaN -> UNCERTAIN + status)
    code[e] = z < A.lo ? NOSCOPE_R_NEG : (z > A.hi ? NOSCOPE_R_POS : NOSCOPE_R_UNC);
    if (in) {
      nneg += code[e] == NOSCOPE_R_NEG;
      npos += code[e] == NOSCOPE_R_POS;
      if (code[e] == NOSCOPE_R_UNC) {
        flags |= 1u << e;
        ++cnt;
      }
      nan |= z != z;
    }
  }
  if (nan) atomicOr(A.status, 2u);
  if (A.route_out) {
    if (full) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = code[4 * q] | (code[4 * q + 1] << 8) | (code[4 * q + 2] << 16) | ((uint32_t)code[4 * q + 3] << 24);
      *reinterpret_cast<uint4*>(A.route_out + base) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
#pragma unroll
      for (int e = 0; e < kScanItems; ++e)
        if (base + e < n) A.route_out[base + e] = code[e];
    }
  }
  if (A.frame_idx) {
#pragma unroll
    for (int e = 0; e < kScanItems; ++e)
      if (base + e < n) {
        const int32_t f = A.frame_idx[base + e];
        if (A.route_pf) A.route_pf[f] = code[e];
        if (A.logits_pf) A.logits_pf[f] = zv[e];
      }
  }
  uint32_t total;
  uint32_t local = block_excl_scan(cnt, warp_sums, &total);
  if (A.counters) {
    if (nneg) atomicAdd(&s_neg, nneg);
    if (npos) atomicAdd(&s_pos, npos);
  }
  {
    uint32_t q = local;
#pragma unroll
    for (int e = 0; e < kScanItems; ++e)
      if (flags & (1u << e)) idx_s[q++] = A.frame_idx ? A.frame_idx[base + e] : (int32_t)(base + e);
  }
  uint64_t excl = tile_lookback(ws, tile, total, &s_excl);  // ends with __syncthreads
  if (A.unc_pos_pf) {
    uint64_t pos = excl + local;
#pragma unroll
    for (int e = 0; e < kScanItems; ++e)
      if (flags & (1u << e)) A.unc_pos_pf[A.frame_idx ? A.frame_idx[base + e] : (int32_t)(base + e)] = (int32_t)pos++;
  }
  store_run(A.unc_out, excl, total, idx_s);
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
              reinterpret_cast<unsigned long long*>(counters), status,
              (int)(((reinterpret_cast<uintptr_t>(logits) | reinterpret_cast<uintptr_t>(route_out)) & 15) == 0)};
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
