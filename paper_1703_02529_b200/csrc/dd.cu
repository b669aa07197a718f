// dd.cu — frame downsampling + difference detector (§5),
// one fused, warp-specialised pass over the source frames.
//
// dd_kernel (persistent, 2 CTAs/SM, 288 threads):
//   * each CTA owns a CONTIGUOUS range of the frames that must be downsampled
//     (checked frames, plus mode-1 anchors), one output row ("band") at a time;
//   * a band = source rows [floor(iH/h), floor((i+1)H/h)) = one contiguous byte
//     range of the frame, fetched by one cp.async.bulk (TMA 1-D engine) into a
//     4-stage shared-memory ring (mbarrier completion, L2 evict-first: every
//     source byte is read exactly once);
//   * warps 0-3 ("V"): vertical byte-column sums of the band, SWAR with two
//     16-bit lanes per 32-bit register (PRMT unpack, 16-byte smem vectors);
//   * warps 4-8 ("H"): box means G = floor((2S+n)/2n) (O1, reading R-1) via a
//     per-column magic reciprocal, the small-frame row store (CNN input), and
//     the exact integer SSD against the anchor row — the reference image kept
//     in smem (mode 0) or frame t-k (mode 1), which this same CTA wrote k
//     frames earlier (it stays L2-resident) — accumulated per thread / per LR
//     block; at frame end the fp64 score (O3) and the disposition (O4);
//   * V and H hand over double-buffered column sums through named barriers,
//     so the two halves of the work overlap band by band;
//   * the few frames whose anchor lies in the previous CTA's range are scored
//     after that CTA publishes its completion flag (no second kernel).
// dd_state_update_kernel carries the last k small frames / labels of a chunk
// into the caller's stream state.
#include "common.cuh"
#include "internal.h"

namespace ns {

uint64_t& launch_counter() {
  static thread_local uint64_t c = 0;
  return c;
}

constexpr int kV = 128;                 // vertical-sum group
constexpr int kHz = 160;                // box-mean / score group (out_w*3 <= 160)
constexpr int kDsThreads = kV + kHz;
constexpr int kDsMaxStages = 8;          // band ring depth: as many as fit 2 CTAs/SM
// named barrier ids (0 = __syncthreads)
constexpr int kBarFull0 = 1, kBarEmpty0 = 3, kBarV = 5, kBarH = 6;

NS_DEV void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
NS_DEV void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
NS_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
NS_DEV void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct DsArgs {
  const uint8_t* frames;
  int64_t frame_pitch;
  int W, H, RB, RBp;  // RB = W*3 bytes per source row, RBp = RB rounded to 16
  int out_w, out_h;
  uint8_t* small;
  int64_t small_pitch;
  NeededSet need;
  int64_t tau0;
  int mode, metric, grid, k, t_skip;
  const uint8_t* ref;
  const float* lr_w;
  float lr_b;
  double delta;
  const uint8_t* ring;  // mode 1 anchors before tau0 (slot (tau-k) % k)
  int64_t ring_pitch;
  double* score;
  uint8_t* disp;
  uint32_t* status;
  unsigned* done;  // [gridDim.x] completion flags, zeroed before launch (mode 1)
  int stage_bytes, fast, rlo, nstages;
};

struct BandInfo {   // per output row i
  int a0;           // aligned byte offset of the band in the frame
  int bytes;        // aligned byte count
  int offrows;      // (misalignment << 16) | nrows
  int bi;           // LR block row
};

NS_DEV int block_of(int i, int n, int g) {
  const int b = i / (n / g);
  return b < g - 1 ? b : g - 1;
}
NS_DEV int64_t frame_of(const NeededSet& s, int64_t m) {  // nres in {1, 2}
  const int64_t p = s.nres == 2 ? (m >> 1) : m;
  return p * s.t_skip + s.res[s.nres == 2 ? (int)(m & 1) : 0] - s.tau0;
}
NS_DEV int64_t range_start(const NeededSet& s, int c, int G) {
  return s.m0 + ((s.m1 - s.m0) * (int64_t)c) / G;
}

struct HzState {  // per box-mean thread
  int t, j, colbase, ncols, bj;
  uint32_t mlo, mhi;
  uint64_t total;
  uint32_t blk;
  int cur_bi;
};

// Frame-end scoring by the H group (all 160 threads call it).
NS_DEV void finish_score(const DsArgs& A, HzState& h, int hz, uint32_t* blk, const uint32_t* blkn,
                         const double* wlr, double* pk, unsigned long long* red, int64_t f,
                         bool active) {
  if (A.metric == 0) {
    unsigned long long v = active ? h.total : 0ull;
    v = warp_sum(v);
    if ((hz & 31) == 0) red[hz >> 5] = v;
    bar_sync(kBarH, kHz);
    if (hz == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < kHz / 32; ++w) s += red[w];
      const double sc = (double)s / (double)(A.out_w * A.out_h * 3);
      A.score[f] = sc;
      A.disp[f] = sc > A.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
    }
    bar_sync(kBarH, kHz);  // red[] reuse
  } else {
    const int gg = A.grid * A.grid;
    if (active && h.cur_bi >= 0 && h.blk) atomicAdd(&blk[h.cur_bi * A.grid + h.bj], h.blk);
    bar_sync(kBarH, kHz);
    for (int q = hz; q < gg; q += kHz) {
      pk[q] = __dmul_rn(wlr[q], (double)blk[q] / (double)blkn[q]);  // w_k * m_k, rounded
      blk[q] = 0u;
    }
    bar_sync(kBarH, kHz);
    if (hz == 0) {
      double z = (double)A.lr_b;
      for (int q = 0; q < gg; ++q) z = __dadd_rn(z, pk[q]);  // fixed order, no FMA
      if (z != z) atomicOr(A.status, 1u);
      A.score[f] = z;
      A.disp[f] = z > A.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
    }
  }
  h.total = 0;
  h.blk = 0;
  h.cur_bi = -1;
}

NS_DEV void ssd_acc(const DsArgs& A, HzState& h, uint32_t d2, int bi, uint32_t* blk) {
  if (A.metric == 0) {
    h.total += d2;
  } else {
    if (bi != h.cur_bi) {
      if (h.cur_bi >= 0 && h.blk) atomicAdd(&blk[h.cur_bi * A.grid + h.bj], h.blk);
      h.cur_bi = bi;
      h.blk = 0;
    }
    h.blk += d2;
  }
}

__global__ void __launch_bounds__(kDsThreads, 2)
dd_kernel(DsArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int gg = A.grid * A.grid;
  const int small_bytes = A.out_w * A.out_h * 3;
  uint8_t* stages = smem;
  uint16_t* cs = reinterpret_cast<uint16_t*>(smem + A.nstages * A.stage_bytes);   // 2 x RBp
  BandInfo* band = reinterpret_cast<BandInfo*>(cs + 2 * A.RBp);
  uint8_t* ref_s = reinterpret_cast<uint8_t*>(band + A.out_h);
  uint32_t* blk = reinterpret_cast<uint32_t*>(ref_s + (A.mode == 0 ? ((small_bytes + 15) & ~15) : 0));
  uint32_t* blkn = blk + ((gg + 1) & ~1);
  double* wlr = reinterpret_cast<double*>(blkn + ((gg + 1) & ~1));
  double* pk = wlr + gg;
  unsigned long long* red = reinterpret_cast<unsigned long long*>(pk + gg);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 8);

  const int tid = threadIdx.x;
  const int64_t mA = range_start(A.need, blockIdx.x, gridDim.x);
  const int64_t mB = range_start(A.need, blockIdx.x + 1, gridDim.x);
  const int64_t my_frames = mB - mA;
  const int64_t total = my_frames * A.out_h;

  // ---- one-time tables
  for (int i = tid; i < A.out_h; i += blockDim.x) {
    const int r0 = (i * A.H) / A.out_h, r1 = ((i + 1) * A.H) / A.out_h;
    const int64_t b0 = (int64_t)r0 * A.RB, b1 = (int64_t)r1 * A.RB;
    const int64_t a0 = b0 & ~(int64_t)15, a1 = (b1 + 15) & ~(int64_t)15;
    band[i].a0 = (int)a0;
    band[i].bytes = (int)(a1 - a0);
    band[i].offrows = ((int)(b0 - a0) << 16) | (r1 - r0);
    band[i].bi = A.metric == 1 ? block_of(i, A.out_h, A.grid) : 0;
  }
  if (A.mode == 0)
    for (int t = tid; t < small_bytes; t += blockDim.x) ref_s[t] = A.ref[t];
  if (A.metric == 1) {
    const int sh = A.out_h / A.grid, sw = A.out_w / A.grid;
    for (int q = tid; q < gg; q += blockDim.x) {
      const int bi = q / A.grid, bj = q % A.grid;
      const int rows = bi < A.grid - 1 ? sh : A.out_h - (A.grid - 1) * sh;
      const int cols = bj < A.grid - 1 ? sw : A.out_w - (A.grid - 1) * sw;
      blk[q] = 0u;
      blkn[q] = (uint32_t)(rows * cols * 3);
      wlr[q] = (double)A.lr_w[q];
    }
  }
  if (tid == 0) {
    for (int s = 0; s < A.nstages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (tid < kV) {
    // =========================================================== V group
    const int vt = tid;
    // producer (vt == 0): issue bands ahead into the ring
    int64_t p_seq = 0, p_m = mA;
    int p_i = 0, p_s = 0;
    const uint64_t pol = policy_evict_first();
    const uint8_t* p_frame = A.frames + frame_of(A.need, p_m) * A.frame_pitch;
    auto issue = [&]() {
      const BandInfo bd = band[p_i];
      mbar_arrive_expect_tx(&full[p_s], (uint32_t)bd.bytes);
      bulk_g2s_evict_first(stages + (size_t)p_s * A.stage_bytes, p_frame + bd.a0, (uint32_t)bd.bytes,
                           &full[p_s], pol);
      ++p_seq;
      p_s = p_s + 1 == A.nstages ? 0 : p_s + 1;
      if (++p_i == A.out_h) {
        p_i = 0;
        ++p_m;
        if (p_m < mB) p_frame = A.frames + frame_of(A.need, p_m) * A.frame_pitch;
      }
    };
    if (vt == 0)
      while (p_seq < A.nstages && p_seq < total) issue();

    int i = 0, s = 0;
    uint32_t ph = 0;
    const int RB16 = A.RB >> 4;
    for (int64_t seq = 0; seq < total; ++seq) {
      const int b = (int)(seq & 1);
      if (seq >= 2) bar_sync(kBarEmpty0 + b, kDsThreads);
      mbar_wait(&full[s], ph);
      const int offrows = band[i].offrows;
      const int nrows = offrows & 0xFFFF, off = offrows >> 16;
      const uint8_t* src = stages + (size_t)s * A.stage_bytes + off;
      uint16_t* dst = cs + b * A.RBp;
      if (A.fast) {
        for (int u = vt; u < RB16; u += kV) {
          const uint4* p = reinterpret_cast<const uint4*>(src) + u;
          uint32_t l0 = 0, h0 = 0, l1 = 0, h1 = 0, l2 = 0, h2 = 0, l3 = 0, h3 = 0;
          for (int r = 0; r < nrows; ++r) {
            const uint4 w = p[(size_t)r * RB16];
            l0 += __byte_perm(w.x, 0u, 0x4240); h0 += __byte_perm(w.x, 0u, 0x4341);
            l1 += __byte_perm(w.y, 0u, 0x4240); h1 += __byte_perm(w.y, 0u, 0x4341);
            l2 += __byte_perm(w.z, 0u, 0x4240); h2 += __byte_perm(w.z, 0u, 0x4341);
            l3 += __byte_perm(w.w, 0u, 0x4240); h3 += __byte_perm(w.w, 0u, 0x4341);
          }
          uint4 o0, o1;
          o0.x = (l0 & 0xFFFFu) | (h0 << 16); o0.y = (l0 >> 16) | (h0 & 0xFFFF0000u);
          o0.z = (l1 & 0xFFFFu) | (h1 << 16); o0.w = (l1 >> 16) | (h1 & 0xFFFF0000u);
          o1.x = (l2 & 0xFFFFu) | (h2 << 16); o1.y = (l2 >> 16) | (h2 & 0xFFFF0000u);
          o1.z = (l3 & 0xFFFFu) | (h3 << 16); o1.w = (l3 >> 16) | (h3 & 0xFFFF0000u);
          reinterpret_cast<uint4*>(dst)[2 * u] = o0;
          reinterpret_cast<uint4*>(dst)[2 * u + 1] = o1;
        }
      } else {
        for (int x = vt; x < A.RB; x += kV) {
          uint32_t sum = 0;
          for (int r = 0; r < nrows; ++r) sum += src[(size_t)r * A.RB + x];
          dst[x] = (uint16_t)sum;
        }
      }
      bar_sync(kBarV, kV);  // every V thread is done with stage s
      if (vt == 0 && p_seq < total) issue();
      bar_arrive(kBarFull0 + b, kDsThreads);
      s = s + 1 == A.nstages ? 0 : s + 1;
      if (s == 0) ph ^= 1u;
      if (++i == A.out_h) i = 0;
    }
    for (int64_t seq = total > 2 ? total - 2 : 0; seq < total; ++seq)
      bar_sync(kBarEmpty0 + (int)(seq & 1), kDsThreads);  // drain the last EMPTY arrivals
    return;
  }

  // ============================================================== H group
  const int hz = tid - kV;
  const int n_out = A.out_w * 3;
  const bool active = hz < n_out;
  HzState h{};
  h.t = hz;
  h.j = hz / 3;
  h.cur_bi = -1;
  if (active) {
    const int c = hz - 3 * h.j;
    const int q0 = (h.j * A.W) / A.out_w, q1 = ((h.j + 1) * A.W) / A.out_w;
    h.colbase = q0 * 3 + c;
    h.ncols = q1 - q0;
    // magic reciprocals of 2n for the two possible band heights (rlo, rlo+1)
    const uint32_t n_lo = (uint32_t)(A.rlo * h.ncols), n_hi = (uint32_t)((A.rlo + 1) * h.ncols);
    h.mlo = (uint32_t)(0x100000000ull / (2ull * n_lo)) + 1u;
    h.mhi = (uint32_t)(0x100000000ull / (2ull * n_hi)) + 1u;
    h.bj = A.metric == 1 ? block_of(h.j, A.out_w, A.grid) : 0;
  }
  const int64_t tau_first = my_frames > 0 ? A.tau0 + frame_of(A.need, mA) : 0;

  int i = 0;
  int64_t m = mA;
  int64_t f = 0, tau = 0;
  bool checked = false, scoring = false, forced = false;
  const uint8_t* anchor = nullptr;
  uint8_t* dstf = nullptr;
  for (int64_t seq = 0; seq < total; ++seq) {
    if (i == 0) {  // frame start
      f = frame_of(A.need, m);
      tau = A.tau0 + f;
      checked = (tau % A.t_skip) == 0;
      forced = A.mode == 1 && checked && tau < A.k;
      scoring = checked && !forced;
      if (scoring && A.mode == 1) {
        const int64_t fa = f - A.k;
        if (fa >= 0) {
          anchor = A.small + fa * A.small_pitch;
          if (tau - A.k < tau_first) scoring = false;  // anchor owned by another CTA: deferred
        } else {
          anchor = A.ring + ((tau - A.k) % A.k) * A.ring_pitch;
        }
      } else if (A.mode == 0) {
        anchor = ref_s;
      }
      dstf = A.small + f * A.small_pitch;
    }
    const int b = (int)(seq & 1);
    bar_sync(kBarFull0 + b, kDsThreads);
    if (active) {
      const BandInfo bd = band[i];
      const int nrows = bd.offrows & 0xFFFF;
      uint32_t av = 0;
      if (scoring) av = anchor[i * n_out + h.t];
      const uint16_t* c0 = cs + b * A.RBp + h.colbase;
      uint32_t S = 0;
      for (int q = 0; q < h.ncols; ++q) S += c0[3 * q];
      const uint32_t n = (uint32_t)nrows * (uint32_t)h.ncols;
      const uint32_t G = __umulhi(2u * S + n, nrows == A.rlo ? h.mlo : h.mhi);
      dstf[i * n_out + h.t] = (uint8_t)G;
      if (scoring) {
        const int d = (int)G - (int)av;
        ssd_acc(A, h, (uint32_t)(d * d), bd.bi, blk);
      }
    }
    bar_arrive(kBarEmpty0 + b, kDsThreads);
    if (++i == A.out_h) {  // frame end
      i = 0;
      if (scoring) {
        finish_score(A, h, hz, blk, blkn, wlr, pk, red, f, active);
      } else if (forced && hz == 0) {
        A.score[f] = __longlong_as_double(0x7FF0000000000000ll);  // +inf
        A.disp[f] = NOSCOPE_FIRED;
      }
      ++m;
    }
  }

  // ---- publish completion, then score deferred frames (mode 1 only)
  if (A.mode != 1) return;
  bar_sync(kBarH, kHz);
  if (hz == 0) {
    __threadfence();
    st_release_u32(&A.done[blockIdx.x], 1u);
  }
  for (int64_t mm = mA; mm < mB; ++mm) {
    const int64_t ff = frame_of(A.need, mm);
    const int64_t tt = A.tau0 + ff;
    if (tt - A.k >= tau_first) break;
    if ((tt % A.t_skip) != 0 || tt < A.k || ff - A.k < 0) continue;
    const int64_t fa = ff - A.k;
    if (hz == 0) {  // wait for the CTA owning the anchor frame
      int c = (int)blockIdx.x - 1;
      while (c > 0 && frame_of(A.need, range_start(A.need, c, gridDim.x)) > fa) --c;
      while (ld_acquire_u32(&A.done[c]) == 0u) {
      }
    }
    bar_sync(kBarH, kHz);
    const uint8_t* G = A.small + ff * A.small_pitch;
    const uint8_t* An = A.small + fa * A.small_pitch;
    if (active)
      for (int r = 0; r < A.out_h; ++r) {
        const int d = (int)G[r * n_out + h.t] - (int)An[r * n_out + h.t];
        ssd_acc(A, h, (uint32_t)(d * d), band[r].bi, blk);
      }
    finish_score(A, h, hz, blk, blkn, wlr, pk, red, ff, active);
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
static size_t ds_smem_bytes(const DsArgs& A, int* stage_bytes_out, int* nstages_out) {
  int stage = 0;
  for (int i = 0; i < A.out_h; ++i) {
    const int r0 = (i * A.H) / A.out_h, r1 = ((i + 1) * A.H) / A.out_h;
    const int64_t b0 = (int64_t)r0 * A.RB, b1 = (int64_t)r1 * A.RB;
    const int64_t a0 = b0 & ~15ll, a1 = (b1 + 15) & ~15ll;
    if ((int)(a1 - a0) > stage) stage = (int)(a1 - a0);
  }
  stage = (stage + 127) & ~127;
  *stage_bytes_out = stage;
  const int gg = A.grid * A.grid;
  const int small_bytes = A.out_w * A.out_h * 3;
  size_t b = 2 * (size_t)A.RBp * sizeof(uint16_t);
  b += (size_t)A.out_h * sizeof(BandInfo);
  b += A.mode == 0 ? (size_t)((small_bytes + 15) & ~15) : 0;   // reference image (mode 0)
  b += 2 * (size_t)((gg + 1) & ~1) * 4;
  b += 2 * (size_t)gg * 8;
  b += 8 * 8 + kDsMaxStages * 8 + 16;
  // ring depth: as many bands as fit with 2 CTAs per SM (227 KB per SM minus the
  // 1 KB per-CTA reservation), at least 2
  const size_t per_cta = (227 * 1024) / 2 - 1024;
  int ns = per_cta > b ? (int)((per_cta - b) / stage) : 0;
  ns = std::max(2, std::min(kDsMaxStages, ns));
  *nstages_out = ns;
  return b + (size_t)ns * stage;
}

size_t dd_flags_bytes() { return (size_t)4 * kNumSMs * 4; }

noscope_status launch_diff_detect(const noscope_dd_config& cfg, const uint8_t* frames,
                                  const noscope_frames_desc& desc, int64_t n, int64_t tau0,
                                  uint8_t* state, uint8_t* small, int64_t small_pitch,
                                  double* score, uint8_t* disp, uint32_t* status, unsigned* flags,
                                  cudaStream_t st, Prof* prof) {
  DsArgs A{};
  A.frames = frames;
  A.frame_pitch = desc.frame_pitch;
  A.W = desc.width;
  A.H = desc.height;
  A.RB = desc.width * 3;
  A.RBp = (A.RB + 15) & ~15;
  A.out_w = cfg.out_w;
  A.out_h = cfg.out_h;
  A.small = small;
  A.small_pitch = small_pitch;
  A.need = make_needed_set(cfg, tau0, n);
  A.tau0 = tau0;
  A.mode = cfg.mode;
  A.metric = cfg.metric;
  A.grid = cfg.metric == 1 ? cfg.grid : 1;
  A.k = cfg.mode == 1 ? cfg.t_diff_frames : 1;
  A.t_skip = cfg.t_skip_frames;
  A.ref = cfg.ref_image;
  A.lr_w = cfg.lr_weights;
  A.lr_b = cfg.lr_bias;
  A.delta = cfg.delta_diff;
  A.ring = state;
  A.ring_pitch = state_ring_pitch(cfg);
  A.score = score;
  A.disp = disp;
  A.status = status;
  A.done = flags;
  A.fast = (A.RB % 16) == 0;
  A.rlo = A.H / A.out_h;
  const size_t smem = ds_smem_bytes(A, &A.stage_bytes, &A.nstages);
  const int64_t frames_needed = A.need.m1 - A.need.m0;
  if (frames_needed > 0) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(dd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_set = true;
    }
    int per_sm = 0;
    NS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dd_kernel, kDsThreads, smem));
    if (per_sm < 1) return NOSCOPE_SHAPE;
    int sms = kNumSMs, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // all CTAs co-resident (deferred scoring waits on earlier CTAs' flags)
    const int grid = (int)std::min<int64_t>(frames_needed, (int64_t)std::min(per_sm, 4) * sms);
    if (cfg.mode == 1) NS_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)grid * 4, st));
    dd_kernel<<<grid, kDsThreads, smem, st>>>(A);
    NS_LAUNCH_CHECK();
    count_launch();
  }
  prof_mark(prof, st);
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
