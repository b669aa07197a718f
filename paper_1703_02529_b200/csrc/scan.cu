// scan.cu — stream compaction ("batch input images"), routing
// and per-frame label resolution.
//
// Compaction of the FIRED frames and of the uncertain logits: one persistent
// two-phase launch each (classify + bitmask + count per contiguous range, grid
// barrier, indices from the bitmask) — see compact_fired_kernel / route_kernel.
// Both outputs are ascending (stable), bit-identical to a serial scan.
//
// Label resolution follows the backward pointers of O8 without pointer
// chasing: among checked frames (tau = p * t_skip) a mode-1 suppression copies
// checked frame p - K, K = ceil(k / t_skip) (the checked frame that frame
// tau - k copies), so labels are a "last resolved value" scan inside each of
// the K residue classes; skipped frames copy their period's checked frame.
// Three launches, a warp per (class, 32-element segment) with the lanes on the
// elements: per-segment summaries, per-class carries (a warp per class), apply.
#include "common.cuh"
#include "internal.h"

namespace ns {

NS_DEV unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
NS_DEV void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------ two-phase bitmask compaction
// Compaction of the FIRED frames (O5) and of the uncertain logits (O7) as one
// persistent cooperative launch each, all G CTAs co-resident, CTA c owning the
// contiguous chunk range [c*C/G, (c+1)*C/G) of 4,096-item warp-chunks:
//   phase 1: stream the range once (coalesced 16-byte loads, 8 in flight per
//            lane), classify every item, write a 1-bit-per-item mask (u16 per 16
//            items) and the side outputs, count the selected items;
//   grid barrier (arrival counter, acquire spin; co-residency from the launch);
//   phase 2: offset = the lower ranges' counts; read only the MASK (1/8 byte per
//            item) and write the ascending indices — each lane owns 128
//            consecutive items, warp scan + block scan give its output position.
// DRAM traffic per item = the item + 1/4 byte of mask (write + read) + 4 bytes per
// selected item: within 1.1x of the algorithmic bytes at 15 % selected.
// Launch shape: one 1,024-thread CTA per SM for both kernels (A/B at 2^30 dispositions /
// 2^28 logits: 0.431-0.433 / 0.418-0.422 ms; 512 threads x 3 (compaction) / x 2 (routing)
// 0.446-0.457 / 0.433-0.446; 768 x 2: 0.431 / 0.422; 256 x 6: 0.477 / 0.441-0.467)
#ifndef NS_MTHREADS
#define NS_MTHREADS 1024
#endif
#ifndef NS_MCPS
#define NS_MCPS 1
#endif
#ifndef NS_RCPS
#define NS_RCPS 1
#endif
constexpr int kMThreads = NS_MTHREADS, kMWarps = kMThreads / 32;
constexpr int kMItems = 16, kMRounds = 4;
constexpr int kMChunk = 32 * kMItems * kMRounds;   // 2048 items per warp-chunk
constexpr int kMHalf = kMChunk / 16;               // mask halfwords per chunk
constexpr int kMLaneWords = kMChunk / 32 / 32;     // phase 2: 32-bit mask words per lane (64 items)
constexpr int kMMaxCtas = 1024;
static_assert(NOSCOPE_FIRED == 2, "SWAR compare below tests bytes == 0x02");

struct MaskWs {
  unsigned* arrive;                // grid-barrier arrivals (zeroed before the launch)
  unsigned long long* cta_count;   // [kMMaxCtas] selected items per CTA range
  uint16_t* masks;                 // [nchunks * kMHalf]: bit e of masks[i / 16] = item i selected
};

size_t compact_ws_bytes(int64_t n) {
  const int64_t nch = (n + kMChunk - 1) / kMChunk;
  return 256 + (size_t)kMMaxCtas * 8 + (((size_t)nch * kMHalf * 2 + 255) & ~size_t(255));
}
static MaskWs mask_ws_of(void* p) {
  uint8_t* b = reinterpret_cast<uint8_t*>(p);
  return MaskWs{reinterpret_cast<unsigned*>(b), reinterpret_cast<unsigned long long*>(b + 256),
                reinterpret_cast<uint16_t*>(b + 256 + kMMaxCtas * 8)};
}

NS_DEV unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
NS_DEV uint4 ld_stream16(const void* p) {   // read-once data: do not keep in L1
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// Per-warp counts of the warps' contiguous sub-ranges -> publish the CTA's sum,
// grid barrier, and return this WARP's exclusive output offset (lower CTAs'
// ranges + lower warps of this CTA).  The last CTA also writes the grand total.
NS_DEV uint64_t grid_exclusive_offset(MaskWs ws, uint32_t mine, int64_t* total_out) {
  __shared__ uint32_t wsum[kMWarps];
  __shared__ uint64_t s_off;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t w = warp_sum(mine);
  if (lane == 0) wsum[warp] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < kMWarps; ++i) t += wsum[i];
    const int c = blockIdx.x, G = gridDim.x;
    st_relaxed(&ws.cta_count[c], (unsigned long long)t);
    __threadfence();
    atomicAdd(ws.arrive, 1u);
    while (ld_acquire_gpu(ws.arrive) < (unsigned)G) {
    }
    uint64_t off = 0;
    for (int q = 0; q < c; ++q) off += ld_relaxed(&ws.cta_count[q]);
    s_off = off;
    if (c == G - 1 && total_out) *total_out = (int64_t)(off + t);
  }
  __syncthreads();
  uint64_t off = s_off;
  for (int i = 0; i < warp; ++i) off += wsum[i];
  return off;
}

// Contiguous chunk sub-range of warp `warp` within the CTA range [ch0, ch1).
NS_DEV void warp_range(int64_t ch0, int64_t ch1, int warp, int64_t* a, int64_t* b) {
  const int64_t len = ch1 - ch0;
  *a = ch0 + len * warp / kMWarps;
  *b = ch0 + len * (warp + 1) / kMWarps;
}

// Phase 2: the selected items of this warp's chunks [wa, wb), ascending, from
// their masks, starting at output position `off`.  Per chunk (2,048 items):
// lane L owns items 64L .. 64L+63 (one 8-byte mask load, prefetched a chunk
// ahead), a warp scan gives each selected item its position in the chunk's run;
// the warp stages the item offsets (u16) in its own shared-memory slice, then
// writes the run with coalesced stores: emit(item, pos) for k = lane, lane + 32, ..
constexpr size_t kMStageBytes = (size_t)kMWarps * kMChunk * 2;   // 4 KB per warp (128 KB per 1,024-thread CTA)

template <class Emit>
NS_DEV void emit_selected(MaskWs ws, int64_t wa, int64_t wb, uint64_t off, uint16_t* stage_all, Emit&& emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* stage = stage_all + (size_t)warp * kMChunk;
  static_assert(kMLaneWords == 2, "one 8-byte mask load per lane");
  auto load = [&](int64_t ch) -> uint2 {
    return ch < wb ? *reinterpret_cast<const uint2*>(ws.masks + (size_t)ch * kMHalf + 4 * lane)
                   : make_uint2(0, 0);
  };
  uint2 nxt = load(wa);
  for (int64_t ch = wa; ch < wb; ++ch) {
    const uint2 m = nxt;
    nxt = load(ch + 1);
    const uint32_t cnt = __popc(m.x) + __popc(m.y);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t q = incl - cnt;
    const uint32_t mw[2] = {m.x, m.y};
#pragma unroll
    for (int j = 0; j < 2; ++j)
      for (uint32_t f = mw[j]; f; f &= f - 1) stage[q++] = (uint16_t)(64 * lane + 32 * j + (__ffs(f) - 1));
    __syncwarp();
    const int64_t item0 = ch * kMChunk;
    for (uint32_t k = lane; k < wtot; k += 32) emit(item0 + stage[k], off + k);
    __syncwarp();                                           // stage reused next chunk
    off += wtot;
  }
}

__global__ void __launch_bounds__(kMThreads, NS_MCPS)
compact_fired_kernel(uint8_t* disp, double* score, int64_t n, int64_t tau0, int t_skip,
                     int32_t* idx_out, int64_t* count_out, MaskWs ws, int vec, int32_t* pos_pf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, c = blockIdx.x;
  const int64_t nch = (n + kMChunk - 1) / kMChunk;
  const int64_t ch0 = nch * c / G, ch1 = nch * (c + 1) / G;
  // ---- phase 1: FIRED masks (after the t_skip rule) and this warp's count
  int64_t wa, wb;
  warp_range(ch0, ch1, warp, &wa, &wb);
  uint32_t mine = 0;
  auto fast_ok = [&](int64_t ch) { return vec && t_skip == 1 && (ch + 1) * kMChunk <= n; };
  auto masks_of = [&](const uint4 (&v)[kMRounds], int64_t ch) {
    uint16_t* mk = ws.masks + (size_t)ch * kMHalf + lane;
#pragma unroll
    for (int r = 0; r < kMRounds; ++r) {   // SWAR: FIRED bytes -> bits (byte e -> bit e)
      const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        m |= (((__vcmpeq4(w[j], 0x02020202u) & 0x01010101u) * 0x01020408u) >> 24) << (4 * j);
      mk[r * 32] = (uint16_t)m;
      mine += __popc(m);
    }
  };
  int64_t ch = wa;
  for (; ch + 1 < wb && fast_ok(ch + 1); ch += 2) {   // two chunks (8 loads per lane) in flight
    uint4 v[2][kMRounds];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int r = 0; r < kMRounds; ++r) v[c][r] = ld_stream16(disp + (ch + c) * kMChunk + r * 512 + lane * 16);
#pragma unroll
    for (int c = 0; c < 2; ++c) masks_of(v[c], ch + c);
  }
  for (; ch < wb; ++ch) {
    const int64_t base = ch * kMChunk;
    if (fast_ok(ch)) {
      uint4 v[kMRounds];
#pragma unroll
      for (int r = 0; r < kMRounds; ++r) v[r] = ld_stream16(disp + base + r * 512 + lane * 16);
      masks_of(v, ch);
    } else {   // tail, misaligned or t_skip > 1: per item (and the skipped rewrite)
      uint16_t* mk = ws.masks + (size_t)ch * kMHalf + lane;
      for (int r = 0; r < kMRounds; ++r) {
        const int64_t i0 = base + r * 512 + lane * 16;
        uint32_t m = 0;
        int ph = t_skip > 1 ? (int)((tau0 + i0) % t_skip) : 0;
        for (int e = 0; e < kMItems; ++e) {
          const int64_t f = i0 + e;
          if (f < n) {
            if (ph != 0) {
              disp[f] = NOSCOPE_SKIPPED;
              if (score) score[f] = __longlong_as_double(0xFFF0000000000000ll);   // -inf
            } else if (disp[f] == NOSCOPE_FIRED) {
              m |= 1u << e;
            }
          }
          if (t_skip > 1 && ++ph == t_skip) ph = 0;
        }
        mk[r * 32] = (uint16_t)m;
        mine += __popc(m);
      }
    }
  }
  const uint64_t off = grid_exclusive_offset(ws, mine, count_out);
  // ---- phase 2: ascending indices from the masks
  extern __shared__ __align__(16) uint16_t mstage[];
  if (idx_out)
    emit_selected(ws, wa, wb, off, mstage, [&](int64_t i, uint64_t p) {
      idx_out[p] = (int32_t)i;
      if (pos_pf) pos_pf[i] = (int32_t)p;
    });
}

noscope_status launch_compact_fired(const uint8_t* /*disp_in*/, uint8_t* disp, double* score,
                                    int64_t n, int64_t tau0, int t_skip, int32_t* idx_out,
                                    int64_t* count_out, void* scan_ws, cudaStream_t st,
                                    int32_t* pos_pf) {
  const int64_t nch = (n + kMChunk - 1) / kMChunk;
  if (nch == 0) {
    if (count_out) NS_CUDA_TRY(cudaMemsetAsync(count_out, 0, sizeof(int64_t), st));
    return NOSCOPE_OK;
  }
  NS_CUDA_TRY(cudaMemsetAsync(scan_ws, 0, 256, st));   // barrier arrivals
  const int vec = (reinterpret_cast<uintptr_t>(disp) & 15) == 0;
  static DeviceInt occ;
  int per_sm = occ.get();
  if (per_sm == 0) {
    NS_CUDA_TRY(cudaFuncSetAttribute(compact_fired_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kMStageBytes));
    NS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compact_fired_kernel, kMThreads,
                                                              kMStageBytes));
    per_sm = std::max(1, per_sm);
    occ.set(per_sm);
  }
  int sms = kNumSMs;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device());
  // persistent and co-resident (the grid barrier): at most the resident CTA count
  const int grid = (int)std::min<int64_t>({nch, (int64_t)per_sm * sms, (int64_t)kMMaxCtas});
  NS_CUDA_TRY(launch_cooperative(compact_fired_kernel, grid, kMThreads, kMStageBytes, st, disp, score, n, tau0, t_skip,
                                 idx_out, count_out, mask_ws_of(scan_ws), vec, pos_pf));
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

// ------------------------------------------------------------ routing
// Same two-phase structure over the fired logits (count from the device):
// phase 1 reads each logit once (float4 loads), writes its route code (compact
// and/or per frame via frame_idx), counts NEG / POS, marks UNCERTAIN in the mask;
// phase 2 writes the uncertain frame indices (and per-frame list positions).
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

NS_DEV uint8_t route_code(float z, float lo, float hi) {
  // NEG iff z < lo, POS iff z > hi, else UNCERTAIN (R-5; NaN -> UNCERTAIN + status)
  return z < lo ? NOSCOPE_R_NEG : (z > hi ? NOSCOPE_R_POS : NOSCOPE_R_UNC);
}

__global__ void __launch_bounds__(kMThreads, NS_RCPS)
route_kernel(RouteArgs A, MaskWs ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, c = blockIdx.x;
  const int64_t n = A.n_dev ? min(*A.n_dev, A.n_max) : A.n_max;
  const int64_t nch = (n + kMChunk - 1) / kMChunk;
  const int64_t ch0 = nch * c / G, ch1 = nch * (c + 1) / G;
  int64_t wa, wb;
  warp_range(ch0, ch1, warp, &wa, &wb);
  uint32_t mine = 0, nneg = 0, npos = 0, nan = 0;
  for (int64_t ch = wa; ch < wb; ++ch) {
    const int64_t base = ch * kMChunk;
    uint16_t* mk = ws.masks + (size_t)ch * kMHalf + lane;
    const bool fast = A.vec && base + kMChunk <= n;
#pragma unroll 1
    for (int r = 0; r < kMRounds; ++r) {
      const int64_t i0 = base + r * 512 + lane * 16;
      float z[kMItems];
      if (fast) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = ld_stream16(A.logits + i0 + 4 * q);
          z[4 * q] = __uint_as_float(v.x);
          z[4 * q + 1] = __uint_as_float(v.y);
          z[4 * q + 2] = __uint_as_float(v.z);
          z[4 * q + 3] = __uint_as_float(v.w);
        }
      } else {
#pragma unroll
        for (int e = 0; e < kMItems; ++e) z[e] = i0 + e < n ? A.logits[i0 + e] : 0.f;
      }
      uint32_t m = 0, w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int e = 0; e < kMItems; ++e) {
        const uint32_t code = route_code(z[e], A.lo, A.hi);
        w[e >> 2] |= code << (8 * (e & 3));
        if (i0 + e < n) {
          nneg += code == NOSCOPE_R_NEG;
          npos += code == NOSCOPE_R_POS;
          m |= (uint32_t)(code == NOSCOPE_R_UNC) << e;
          nan |= z[e] != z[e];
        }
      }
      mk[r * 32] = (uint16_t)m;
      mine += __popc(m);
      if (A.route_out) {
        if (fast) {
          *reinterpret_cast<uint4*>(A.route_out + i0) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
          for (int e = 0; e < kMItems; ++e)
            if (i0 + e < n) A.route_out[i0 + e] = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
        }
      }
      if (A.frame_idx) {
        for (int e = 0; e < kMItems; ++e)
          if (i0 + e < n) {
            const int32_t f = A.frame_idx[i0 + e];
            if (A.route_pf) A.route_pf[f] = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
            if (A.logits_pf) A.logits_pf[f] = z[e];
          }
      }
    }
  }
  if (nan) atomicOr(A.status, 2u);
  if (A.counters) {
    nneg = warp_sum(nneg);
    npos = warp_sum(npos);
    if (lane == 0 && (nneg | npos)) {
      atomicAdd(&A.counters[0], (unsigned long long)nneg);
      atomicAdd(&A.counters[1], (unsigned long long)npos);
    }
  }
  if (nch == 0) {   // no items: the count is still written
    if (c == 0 && threadIdx.x == 0) *A.n_unc = 0;
    return;
  }
  const uint64_t off = grid_exclusive_offset(ws, mine, A.n_unc);
  extern __shared__ __align__(16) uint16_t mstage[];
  emit_selected(ws, wa, wb, off, mstage, [&](int64_t i, uint64_t p) {
    const int32_t f = A.frame_idx ? A.frame_idx[i] : (int32_t)i;
    A.unc_out[p] = f;
    if (A.unc_pos_pf) A.unc_pos_pf[f] = (int32_t)p;
  });
}

noscope_status launch_route(noscope_route r, const float* logits, const int64_t* n_dev,
                            int64_t n_max, const int32_t* frame_idx, uint8_t* route_out,
                            uint8_t* route_pf, int32_t* unc_out, int64_t* n_unc,
                            int32_t* unc_pos_pf, float* logits_pf, uint64_t* counters,
                            void* scan_ws, uint32_t* status, cudaStream_t st) {
  const int64_t nch = std::max<int64_t>(1, (n_max + kMChunk - 1) / kMChunk);
  NS_CUDA_TRY(cudaMemsetAsync(scan_ws, 0, 256, st));   // barrier arrivals
  RouteArgs A{r.lo_logit, r.hi_logit, logits, n_dev, n_max, frame_idx, route_out, route_pf,
              unc_out, n_unc, unc_pos_pf, logits_pf,
              reinterpret_cast<unsigned long long*>(counters), status,
              (int)(((reinterpret_cast<uintptr_t>(logits) | reinterpret_cast<uintptr_t>(route_out)) & 15) == 0)};
  static DeviceInt occ;
  int per_sm = occ.get();
  if (per_sm == 0) {
    NS_CUDA_TRY(cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMStageBytes));
    NS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_kernel, kMThreads, kMStageBytes));
    per_sm = std::max(1, per_sm);
    occ.set(per_sm);
  }
  int sms = kNumSMs;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device());
  // n_max bounds the device count: every CTA a grid of this size could need is launched
  const int grid = (int)std::min<int64_t>({nch, (int64_t)per_sm * sms, (int64_t)kMMaxCtas});
  NS_CUDA_TRY(launch_cooperative(route_kernel, grid, kMThreads, kMStageBytes, st, A, mask_ws_of(scan_ws)));
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

// One warp per (class r, segment s) of 32 checked elements, lane = element: the
// element values are read in one instruction, and "copy the predecessor" (kNone)
// is resolved by a warp scan of the last defined value.
NS_DEV uint8_t warp_last_defined(uint8_t v, int lane, bool inclusive) {
  // returns, per lane, the value of the nearest lane <= lane (inclusive) or < lane
  // (exclusive) whose v != kNone, else kNone
  const unsigned def = __ballot_sync(0xffffffffu, v != kNone);
  const unsigned upto = inclusive ? (lane == 31 ? 0xffffffffu : ((1u << (lane + 1)) - 1)) : ((1u << lane) - 1);
  const unsigned m = def & upto;
  const int src = m ? 31 - __clz(m) : 0;
  const uint8_t w = (uint8_t)__shfl_sync(0xffffffffu, (int)v, src);
  return m ? w : kNone;
}

__global__ void labels_summary_kernel(LabArgs A) {
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wg >= (int64_t)A.K * A.nseg) return;
  const int r = (int)(wg / A.nseg), s = (int)(wg % A.nseg);
  const int64_t e = (int64_t)(s * kSeg + lane) * A.K + r;
  uint8_t v = kNone;
  if (e < A.nc) v = checked_value(A, (A.p_first + e) * A.t_skip - A.tau0);
  const uint8_t last = warp_last_defined(v, 31, true);   // lane 31's inclusive view = the segment's last value
  if (lane == 0) A.summary[wg] = last;
}

// carry into segment s of class r = the last defined summary of segments < s (one
// warp per class walks its segments 32 at a time), else the class head's
// predecessor from the label history; stored after the summaries.
__global__ void labels_carry_kernel(LabArgs A) {
  const int r = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= A.K) return;
  uint8_t* carry = A.summary + (int64_t)A.K * A.nseg;
  uint8_t run = kNone;
  for (int s0 = 0; s0 < A.nseg; s0 += 32) {
    const int s = s0 + lane;
    const uint8_t v = s < A.nseg ? A.summary[(int64_t)r * A.nseg + s] : kNone;
    uint8_t c = warp_last_defined(v, lane, false);    // segments s0 .. s-1
    if (c == kNone) c = run;
    if (s < A.nseg) carry[(int64_t)r * A.nseg + s] = c;
    const uint8_t tail = warp_last_defined(v, 31, true);
    if (tail != kNone) run = tail;
  }
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
  const int64_t wg = t >> 5;
  const int lane = (int)(t & 31);
  if (wg >= (int64_t)A.K * A.nseg) return;
  const int r = (int)(wg / A.nseg), s = (int)(wg % A.nseg);
  uint8_t carry = kNone;
  if (A.mode == 1) {
    carry = A.summary[(int64_t)A.K * A.nseg + wg];
    if (carry == kNone) {
      const int64_t p_pred = A.p_first + r - A.K;  // predecessor of the class head
      carry = p_pred >= 0 ? hist_label(A, p_pred * A.t_skip) : 0;
    }
  }
  const int64_t e = (int64_t)(s * kSeg + lane) * A.K + r;
  const bool in = e < A.nc;
  const int64_t tau = (A.p_first + e) * A.t_skip;
  const int64_t f = tau - A.tau0;
  uint8_t v = in ? checked_value(A, f) : kNone;
  const uint8_t prev = warp_last_defined(v, lane, true);   // suppressed elements copy the last defined one
  if (!in) return;
  v = prev != kNone ? prev : carry;
  const uint8_t d = A.disp[f];
  A.labels[f] = v;
  if (A.route_out) A.route_out[f] = d == NOSCOPE_FIRED ? A.route_pf[f] : (uint8_t)NOSCOPE_R_SUPP;
  for (int q = 1; q < A.t_skip && f + q < A.n; ++q) {
    A.labels[f + q] = v;
    if (A.route_out) A.route_out[f + q] = NOSCOPE_R_SKIP;
  }
}

size_t labels_ws_bytes(int64_t n) { return (size_t)(2 * (n / kSeg + 4096)); }   // summaries + carries

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
  const int64_t warps = (int64_t)A.K * A.nseg;
  const int blocks = (int)std::max<int64_t>(1, (warps * 32 + 255) / 256);
  if (cfg.mode == 1 && warps > 0) {
    labels_summary_kernel<<<blocks, 256, 0, st>>>(A);
    NS_LAUNCH_CHECK();
    labels_carry_kernel<<<(int)((A.K * 32 + 255) / 256), 256, 0, st>>>(A);
    NS_LAUNCH_CHECK();
    count_launch(2);
  }
  labels_apply_kernel<<<blocks, 256, 0, st>>>(A);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

}  // namespace ns
