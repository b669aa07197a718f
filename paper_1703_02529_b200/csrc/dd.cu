// dd.cu — frame downsampling + difference detector (§5),
// one fused, warp-specialised pass over the source frames.
//
// dd_kernel (persistent, normally 1 CTA/SM):
//   * each CTA owns a CONTIGUOUS range of the frames that must be downsampled
//     (checked frames, plus mode-1 anchors), one output row ("band") at a time;
//   * a band = source rows [floor(iH/h), floor((i+1)H/h)) = one contiguous byte
//     range of the frame, fetched by one cp.async.bulk (TMA 1-D engine; every
//     source byte is read exactly once) into a shared-memory
//     ring issued by one producer thread (warp 0);
//   * bands are dealt round-robin to NG worker GROUPS (band i -> group i % NG),
//     each with its own ring of stages (full/empty mbarriers), so groups work on
//     different bands at once and no CTA-wide barrier sits on the path;
//   * a group = NS worker warps, one per column SEGMENT of the output row (a run
//     of output pixels and the source bytes under them).  A worker warp forms the
//     vertical byte-column sums of its segment (SWAR, two 16-bit lanes per word,
//     PRMT unpack of 16-byte smem vectors) into a warp-private buffer, releases
//     the stage, then each lane owns one output value (pixel j, channel c): the
//     box mean G = floor((2S+n)/2n) (O1, reading R-1) via an exact magic
//     reciprocal, the small-frame store (CNN input) and the exact integer SSD
//     against the anchor — the reference image in smem (mode 0) or frame t-k
//     (mode 1), which the SAME lane wrote k frames earlier (program order, no
//     fence) — accumulated per LR block (u64 smem atomics, once per block row);
//   * warp 1 scores each frame when all workers have arrived on its frame
//     barrier: fp64 block means, w_k*m_k and the fixed-order sum (O3), the
//     disposition (O4); per-frame block sums are double-buffered by frame parity;
//   * the few frames whose anchor lies in the previous CTA's range are scored
//     after that CTA publishes its completion flag (no second kernel).
// dd_state_update_kernel carries the last k small frames / labels of a chunk
// into the caller's stream state.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace ns {

uint64_t& launch_counter() {
  static thread_local uint64_t c = 0;
  return c;
}

constexpr int kDsMaxStages = 128;       // all groups' rings together (deep rings for small bands)
constexpr int kDsMaxGroups = 5;
constexpr int kDsMaxWorkers = 20;       // NG * NS worker warps (launch bound: 22 warps)
constexpr int kDsMaxThreads = (2 + kDsMaxWorkers) * 32;
constexpr int kBarEnd = 1;              // named barrier: all warps but the producer
constexpr int kDsHeadBytes = 2 * kDsMaxStages * 8 + 4 * 8 + 32;  // mbarriers: full/empty, fdone/bfree[2]

// mbarrier phase wait without a suspend-time hint (spins on try_wait; the band
// hand-offs are short, so no sleep/wake latency on the critical path)
NS_DEV void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar), done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
NS_DEV void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct DsArgs {
  const uint8_t* frames;
  int64_t frame_pitch;
  int W, H, RB;  // RB = W*3 bytes per source row
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
  int stage_bytes, fast, rlo;
  int ng, ns, nsg;  // worker groups, segments (warps) per group, ring stages per group
  int cs_stride;    // u16 words of column sums per worker warp (multiple of 8)
  // dynamic smem byte offsets (host-planned, ds_plan)
  int off_ref, off_blkn, off_blk, off_wlr, off_cs, off_stages;
  FiredQueue fq;    // fq.q != null: append fired frames (overlapped cascade)
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

// Column segment of worker `seg` (host and device agree on this split): output
// pixels [j0, j1), source bytes of a row [xb, xb + span) (xb 16-aligned on the
// vector path; span a multiple of 16 there).
struct Seg {
  int j0, j1, xb, span;
};
__host__ __device__ inline Seg segment_of(int seg, int ns, int out_w, int W, bool fast) {
  const int P = (out_w + ns - 1) / ns;
  Seg g;
  g.j0 = min(seg * P, out_w);
  g.j1 = min(g.j0 + P, out_w);
  const int xs = (int)(((int64_t)g.j0 * W) / out_w) * 3;
  const int xe = (int)(((int64_t)g.j1 * W) / out_w) * 3;
  if (fast) {
    g.xb = xs & ~15;
    g.span = ((xe + 15) & ~15) - g.xb;
  } else {
    g.xb = xs;
    g.span = xe - xs;
  }
  if (g.j1 <= g.j0) g.span = 0;
  return g;
}

// Per-frame role flags, identical in every role (O4 order).
struct FrameCtx {
  int64_t f, tau;
  bool scoring, forced;
  const uint8_t* anchor;  // mode 1: global frame t-k (small buffer or state ring)
};
NS_DEV FrameCtx frame_ctx(const DsArgs& A, int64_t m, int64_t tau_first) {
  FrameCtx c;
  c.f = frame_of(A.need, m);
  c.tau = A.tau0 + c.f;
  const bool checked = A.t_skip == 1 || (c.tau % A.t_skip) == 0;
  c.forced = A.mode == 1 && checked && c.tau < A.k;
  c.scoring = checked && !c.forced;
  c.anchor = nullptr;
  if (c.scoring && A.mode == 1) {
    const int64_t fa = c.f - A.k;
    if (fa >= 0) {
      c.anchor = A.small + fa * A.small_pitch;
      if (c.tau - A.k < tau_first) c.scoring = false;  // anchor owned by another CTA: deferred
    } else {
      c.anchor = A.ring + ((c.tau - A.k) % A.k) * A.ring_pitch;
    }
  }
  return c;
}

// Append fired frame f to the queue (scorer lane 0).  The frame's small image was
// written by this CTA's worker warps before they arrived on its frame barrier, which
// this thread has waited on: the fence + release store publish it at gpu scope.
NS_DEV void fq_push(const DsArgs& A, int64_t f) {
  if (!A.fq.q) return;
  const unsigned long long p = atomicAdd(A.fq.count, 1ull);
  st_release_s32(A.fq.q + p, (int32_t)f);   // release: cumulative over the observed writes
}
// Every entry of this CTA is published (scorer lane 0, after its last push).
NS_DEV void fq_finish(const DsArgs& A) {
  if (!A.fq.q) return;
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.fq.done) : "memory");
}

// Score of one frame from its per-block SSDs (one warp): O3, fixed order.
NS_DEV void score_frame(const DsArgs& A, uint32_t* blk, const uint32_t* blkn,
                        const double* wlr, double* pk, int64_t f, int lane) {
  if (A.metric == 0) {
    if (lane == 0) {
      const double sc = (double)blk[0] / (double)(A.out_w * A.out_h * 3);
      blk[0] = 0u;
      A.score[f] = sc;
      A.disp[f] = sc > A.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
      if (sc > A.delta) fq_push(A, f);
    }
  } else {
    const int gg = A.grid * A.grid;
    for (int q = lane; q < gg; q += 32) {
      pk[q] = __dmul_rn(wlr[q], (double)blk[q] / (double)blkn[q]);  // w_k * m_k, rounded
      blk[q] = 0u;
    }
    __syncwarp();
    if (lane == 0) {
      double z = (double)A.lr_b;
      for (int q = 0; q < gg; ++q) z = __dadd_rn(z, pk[q]);  // fixed order, no FMA
      if (z != z) atomicOr(A.status, 1u);
      A.score[f] = z;
      A.disp[f] = z > A.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
      if (z > A.delta) fq_push(A, f);
    }
  }
  __syncwarp();
}

// Warp-wide flush of the lanes' block-row SSDs: one reduction + one u32 smem atomic
// per LR block column the warp covers (bi is warp-uniform: all lanes are on one band).
NS_DEV void flush_blocks(uint32_t* b, int bi, int grid, int bj, int bj_lo, int bj_hi, uint32_t acc,
                         int lane) {
  for (int q = bj_lo; q <= bj_hi; ++q) {
    const uint32_t v = __reduce_add_sync(0xffffffffu, bj == q ? acc : 0u);
    if (lane == 0 && v) atomicAdd(&b[bi * grid + q], v);
  }
}

// Vertical byte-column sums of one band (fast path), SWAR: two 16-bit lanes per
// word (PRMT unpack), two source rows folded per IADD3.  RLO > 0: rows = RLO or
// RLO + 1 (compile-time unrolled); STRIDE16 > 0: compile-time row stride in uint4.
template <int RLO, int STRIDE16>
NS_DEV void vsum(const uint4* p, int nrows, int stride16, uint32_t (&l)[4], uint32_t (&h)[4]) {
  const int st = STRIDE16 > 0 ? STRIDE16 : stride16;
#define NS_ACC1(V_)                                                                   \
  l[0] += __byte_perm(V_.x, 0u, 0x4240); h[0] += __byte_perm(V_.x, 0u, 0x4341);        \
  l[1] += __byte_perm(V_.y, 0u, 0x4240); h[1] += __byte_perm(V_.y, 0u, 0x4341);        \
  l[2] += __byte_perm(V_.z, 0u, 0x4240); h[2] += __byte_perm(V_.z, 0u, 0x4341);        \
  l[3] += __byte_perm(V_.w, 0u, 0x4240); h[3] += __byte_perm(V_.w, 0u, 0x4341);
#define NS_ACC2(P_, Q_)                                                                        \
  l[0] += __byte_perm(P_.x, 0u, 0x4240) + __byte_perm(Q_.x, 0u, 0x4240);                       \
  h[0] += __byte_perm(P_.x, 0u, 0x4341) + __byte_perm(Q_.x, 0u, 0x4341);                       \
  l[1] += __byte_perm(P_.y, 0u, 0x4240) + __byte_perm(Q_.y, 0u, 0x4240);                       \
  h[1] += __byte_perm(P_.y, 0u, 0x4341) + __byte_perm(Q_.y, 0u, 0x4341);                       \
  l[2] += __byte_perm(P_.z, 0u, 0x4240) + __byte_perm(Q_.z, 0u, 0x4240);                       \
  h[2] += __byte_perm(P_.z, 0u, 0x4341) + __byte_perm(Q_.z, 0u, 0x4341);                       \
  l[3] += __byte_perm(P_.w, 0u, 0x4240) + __byte_perm(Q_.w, 0u, 0x4240);                       \
  h[3] += __byte_perm(P_.w, 0u, 0x4341) + __byte_perm(Q_.w, 0u, 0x4341);
  if (RLO > 0) {
#pragma unroll
    for (int r = 0; r + 1 < RLO; r += 2) {
      const uint4 a = p[r * st], b = p[(r + 1) * st];
      NS_ACC2(a, b)
    }
    if (RLO & 1) {
      const uint4 a = p[(RLO - 1) * st];
      if (nrows > RLO) {
        const uint4 b = p[RLO * st];
        NS_ACC2(a, b)
      } else {
        NS_ACC1(a)
      }
    } else if (nrows > RLO) {
      const uint4 a = p[RLO * st];
      NS_ACC1(a)
    }
  } else {
    int r = 0;
    for (; r + 1 < nrows; r += 2) {
      const uint4 a = p[r * st], b = p[(r + 1) * st];
      NS_ACC2(a, b)
    }
    if (r < nrows) {
      const uint4 a = p[r * st];
      NS_ACC1(a)
    }
  }
#undef NS_ACC1
#undef NS_ACC2
}

// RLO / CLO > 0: the band height / box width is RLO or RLO+1 rows / CLO or CLO+1
// pixels (compile-time unrolled loops); STRIDE16 > 0: source row stride in uint4.
// <0, 0, 0> is the generic kernel.
template <int RLO, int CLO, int STRIDE16>
__global__ void __launch_bounds__(kDsMaxThreads, 1)
dd_kernel(DsArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int gg = A.grid * A.grid;
  const int gg2 = (gg + 1) & ~1;
  const int small_bytes = A.out_w * A.out_h * 3;
  const int n_out = A.out_w * 3;
  const int nstages = A.ng * A.nsg;
  const int nworkers = A.ng * A.ns;
  // fixed-offset head (mbarriers, band table), then the host-planned variable part
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kDsMaxStages;
  uint64_t* fdone = empty + kDsMaxStages;   // [2] all workers finished frame m (parity m & 1)
  uint64_t* bfree = fdone + 2;              // [2] scorer released the block sums of frame m
  BandInfo* band = reinterpret_cast<BandInfo*>(smem + kDsHeadBytes);
  uint8_t* ref_s = smem + A.off_ref;
  uint32_t* blkn = reinterpret_cast<uint32_t*>(smem + A.off_blkn);
  uint32_t* blk = reinterpret_cast<uint32_t*>(smem + A.off_blk);
  double* wlr = reinterpret_cast<double*>(smem + A.off_wlr);
  double* pk = wlr + gg2;
  uint16_t* csbuf = reinterpret_cast<uint16_t*>(smem + A.off_cs);
  uint8_t* stages = smem + A.off_stages;
  (void)nstages;
  (void)nworkers;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t mA = range_start(A.need, blockIdx.x, gridDim.x);
  const int64_t mB = range_start(A.need, blockIdx.x + 1, gridDim.x);
  const int64_t my_frames = mB - mA;

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
  for (int q = tid; q < 2 * gg2; q += blockDim.x) blk[q] = 0u;
  if (A.metric == 1) {
    const int sh = A.out_h / A.grid, sw = A.out_w / A.grid;
    for (int q = tid; q < gg; q += blockDim.x) {
      const int bi = q / A.grid, bj = q % A.grid;
      const int rows = bi < A.grid - 1 ? sh : A.out_h - (A.grid - 1) * sh;
      const int cols = bj < A.grid - 1 ? sw : A.out_w - (A.grid - 1) * sw;
      blkn[q] = (uint32_t)(rows * cols * 3);
      wlr[q] = (double)A.lr_w[q];
    }
  }
  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], (uint32_t)A.ns);
    }
    for (int p = 0; p < 2; ++p) {
      mbar_init(&fdone[p], (uint32_t)nworkers);
      mbar_init(&bfree[p], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t tau_first = my_frames > 0 ? A.tau0 + frame_of(A.need, mA) : 0;

  if (warp == 0) {
    // ======================================================= producer
    if (lane != 0) return;
    int gs[kDsMaxGroups] = {};
    uint32_t gph[kDsMaxGroups] = {};
    int64_t issued[kDsMaxGroups] = {};
    for (int64_t m = mA; m < mB; ++m) {
      const uint8_t* fr = A.frames + frame_of(A.need, m) * A.frame_pitch;
      int g = 0;
      for (int i = 0; i < A.out_h; ++i) {
        const BandInfo bd = band[i];
        const int st = g * A.nsg + gs[g];
        if (issued[g] >= A.nsg) mbar_wait(&empty[st], gph[g] ^ 1u);
        mbar_arrive_expect_tx(&full[st], (uint32_t)bd.bytes);
        bulk_g2s(stages + (size_t)st * A.stage_bytes, fr + bd.a0, (uint32_t)bd.bytes, &full[st]);
        ++issued[g];
        if (++gs[g] == A.nsg) {
          gs[g] = 0;
          gph[g] ^= 1u;
        }
        if (++g == A.ng) g = 0;
      }
    }
    return;
  }

  if (warp == 1) {
    // ========================================================= scorer
    for (int64_t m = mA; m < mB; ++m) {
      const int64_t lm = m - mA;
      mbar_wait(&fdone[lm & 1], (uint32_t)((lm >> 1) & 1));
      const FrameCtx c = frame_ctx(A, m, tau_first);
      uint32_t* b = blk + (lm & 1) * gg2;
      if (c.scoring) {
        score_frame(A, b, blkn, wlr, pk, c.f, lane);
      } else if (c.forced && lane == 0) {
        A.score[c.f] = __longlong_as_double(0x7FF0000000000000ll);  // +inf
        A.disp[c.f] = NOSCOPE_FIRED;
        fq_push(A, c.f);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bfree[lm & 1]);
    }
  } else {
    // ========================================================= workers
    const int wk = warp - 2;
    const int grp = wk / A.ns, seg = wk % A.ns;
    const Seg sg = segment_of(seg, A.ns, A.out_w, A.W, A.fast != 0);
    uint16_t* csw = csbuf + (size_t)wk * A.cs_stride;
    const int nout = (sg.j1 - sg.j0) * 3;
    const bool active = lane < nout;
    const int tg = sg.j0 * 3 + lane;  // output value (row-local index) owned by this lane
    int colbase = 0, ncols = 0, bj = 0;
    int hoff[4] = {0, 0, 0, 0};  // u16 slots of columns colbase + 3q, q < 4
    uint32_t mlo = 0, mhi = 0;
    if (active) {
      const int j = tg / 3, c = tg - 3 * j;
      const int q0 = (int)(((int64_t)j * A.W) / A.out_w), q1 = (int)(((int64_t)(j + 1) * A.W) / A.out_w);
      colbase = q0 * 3 + c - sg.xb;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int x = colbase + 3 * q;
        hoff[q] = A.fast ? ((x & ~3) | ((x & 1) << 1) | ((x >> 1) & 1)) : x;
      }
      ncols = q1 - q0;
      // magic reciprocals of 2n for the two possible band heights (rlo, rlo+1)
      const uint32_t n_lo = (uint32_t)(A.rlo * ncols), n_hi = (uint32_t)((A.rlo + 1) * ncols);
      mlo = (uint32_t)(0x100000000ull / (2ull * n_lo)) + 1u;
      mhi = (uint32_t)(0x100000000ull / (2ull * n_hi)) + 1u;
      bj = A.metric == 1 ? block_of(j, A.out_w, A.grid) : 0;
    }
    // LR block columns this warp covers (warp-uniform)
    const int bj_lo = A.metric == 1 && sg.j1 > sg.j0 ? block_of(sg.j0, A.out_w, A.grid) : 0;
    const int bj_hi = A.metric == 1 && sg.j1 > sg.j0 ? block_of(sg.j1 - 1, A.out_w, A.grid) : 0;
    const int nvec = sg.span >> 4;
    const int RB16 = A.RB >> 4;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t m = mA; m < mB; ++m) {
      const int64_t lm = m - mA;
      const FrameCtx c = frame_ctx(A, m, tau_first);
      const uint8_t* anchor = A.mode == 0 ? ref_s : c.anchor;
      uint8_t* dstf = A.small + c.f * A.small_pitch;
      if (lm >= 2) mbar_wait(&bfree[lm & 1], (uint32_t)(((lm >> 1) - 1) & 1));
      uint32_t* b = blk + (lm & 1) * gg2;
      uint32_t acc = 0u;
      int cur_bi = -1;
      // anchor values are fetched one band ahead (t-k frames come from L2)
      uint32_t av_next = (c.scoring && active && grp < A.out_h) ? anchor[grp * n_out + tg] : 0u;
      for (int i = grp; i < A.out_h; i += A.ng) {
        const uint32_t av = av_next;
        if (c.scoring && active && i + A.ng < A.out_h) av_next = anchor[(i + A.ng) * n_out + tg];
        const int offrows = band[i].offrows;
        const int nrows = offrows & 0xFFFF, off = offrows >> 16;
        const uint8_t* src = stages + (size_t)(grp * A.nsg + s) * A.stage_bytes + off;
        mbar_wait_spin(&full[grp * A.nsg + s], ph);
        if (A.fast) {
          const uint4* p0 = reinterpret_cast<const uint4*>(src + sg.xb);
          for (int u = lane; u < nvec; u += 32) {
            uint32_t l[4] = {0u, 0u, 0u, 0u}, h[4] = {0u, 0u, 0u, 0u};
            vsum<RLO, STRIDE16>(p0 + u, nrows, RB16, l, h);
            // stored as computed: u16 slot of column byte b is b with bits 0 and 1 swapped
            // (l_j = columns 4j, 4j+2; h_j = columns 4j+1, 4j+3); see hoff below
            reinterpret_cast<uint4*>(csw)[2 * u] = make_uint4(l[0], h[0], l[1], h[1]);
            reinterpret_cast<uint4*>(csw)[2 * u + 1] = make_uint4(l[2], h[2], l[3], h[3]);
          }
        } else {
          const uint8_t* p0 = src + sg.xb;
          for (int x = lane; x < sg.span; x += 32) {
            uint32_t sum = 0;
            for (int r = 0; r < nrows; ++r) sum += p0[(size_t)r * A.RB + x];
            csw[x] = (uint16_t)sum;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[grp * A.nsg + s]);  // stage consumed
        if (++s == A.nsg) {
          s = 0;
          ph ^= 1u;
        }
        uint32_t dd2 = 0u;
        if (active) {
          // column colbase + 3q sits at hoff[q & 3] + 12 * (q >> 2) (12 = 0 mod 4 keeps
          // the swapped bits), so every load has a compile-time offset from 4 bases
          uint32_t S = 0;
          if (CLO > 0) {
#pragma unroll
            for (int q = 0; q < CLO; ++q) S += csw[hoff[q & 3] + 12 * (q >> 2)];
            if (ncols > CLO) S += csw[hoff[CLO & 3] + 12 * (CLO >> 2)];
          } else {
            for (int q = 0; q < ncols; q += 4) {
              const int b = 3 * q;
              S += csw[hoff[0] + b];
              if (q + 1 < ncols) S += csw[hoff[1] + b];
              if (q + 2 < ncols) S += csw[hoff[2] + b];
              if (q + 3 < ncols) S += csw[hoff[3] + b];
            }
          }
          const uint32_t n = (uint32_t)nrows * (uint32_t)ncols;
          const uint32_t G = __umulhi(2u * S + n, nrows == A.rlo ? mlo : mhi);
          dstf[i * n_out + tg] = (uint8_t)G;
          const int d = (int)G - (int)av;
          dd2 = (uint32_t)(d * d);
        }
        if (c.scoring) {  // warp-uniform
          const int bi = band[i].bi;
          if (bi != cur_bi) {
            if (cur_bi >= 0) flush_blocks(b, cur_bi, A.grid, bj, bj_lo, bj_hi, acc, lane);
            cur_bi = bi;
            acc = 0u;
          }
          acc += dd2;
        }
        __syncwarp();  // csw reuse by the next band
      }
      if (cur_bi >= 0) flush_blocks(b, cur_bi, A.grid, bj, bj_lo, bj_hi, acc, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&fdone[lm & 1]);
    }
  }

  // ---- publish completion, then score deferred frames (mode 1 only)
  if (A.mode != 1) {
    if (warp == 1 && lane == 0) fq_finish(A);
    return;
  }
  const int nthr = blockDim.x - 32;  // every warp but the producer
  const int et = tid - 32;
  bar_sync(kBarEnd, nthr);
  if (et == 0) {
    __threadfence();
    st_release_u32(&A.done[blockIdx.x], 1u);
  }
  for (int64_t mm = mA; mm < mB; ++mm) {
    const int64_t ff = frame_of(A.need, mm);
    const int64_t tt = A.tau0 + ff;
    if (tt - A.k >= tau_first) break;
    if ((tt % A.t_skip) != 0 || tt < A.k || ff - A.k < 0) continue;
    const int64_t fa = ff - A.k;
    if (et == 0) {  // wait for the CTA owning the anchor frame
      int c = (int)blockIdx.x - 1;
      while (c > 0 && frame_of(A.need, range_start(A.need, c, gridDim.x)) > fa) --c;
      while (ld_acquire_u32(&A.done[c]) == 0u) {
      }
    }
    bar_sync(kBarEnd, nthr);
    if (warp >= 2) {  // same lane -> output mapping as the main loop; few atomics
      const int wk = warp - 2;
      const int grp = wk / A.ns;
      const Seg sg = segment_of(wk % A.ns, A.ns, A.out_w, A.W, A.fast != 0);
      const int tg = sg.j0 * 3 + lane;
      const bool act = lane < (sg.j1 - sg.j0) * 3;
      const int bj = A.metric == 1 && act ? block_of(tg / 3, A.out_w, A.grid) : 0;
      const int bj_lo = A.metric == 1 && sg.j1 > sg.j0 ? block_of(sg.j0, A.out_w, A.grid) : 0;
      const int bj_hi = A.metric == 1 && sg.j1 > sg.j0 ? block_of(sg.j1 - 1, A.out_w, A.grid) : 0;
      const uint8_t* G = A.small + ff * A.small_pitch;
      const uint8_t* An = A.small + fa * A.small_pitch;
      uint32_t acc = 0u;
      int cur_bi = -1;
      constexpr int kB = 8;  // rows loaded per batch (L2 latency overlapped)
      for (int i0 = grp; i0 < A.out_h; i0 += kB * A.ng) {
        int dv[kB];
#pragma unroll
        for (int t = 0; t < kB; ++t) {
          const int i = i0 + t * A.ng;
          dv[t] = act && i < A.out_h ? (int)G[i * n_out + tg] - (int)An[i * n_out + tg] : 0;
        }
#pragma unroll
        for (int t = 0; t < kB; ++t) {
          const int i = i0 + t * A.ng;
          if (i < A.out_h) {  // warp-uniform
            const int bi = band[i].bi;
            if (bi != cur_bi) {
              if (cur_bi >= 0) flush_blocks(blk, cur_bi, A.grid, bj, bj_lo, bj_hi, acc, lane);
              cur_bi = bi;
              acc = 0u;
            }
            acc += (uint32_t)(dv[t] * dv[t]);
          }
        }
      }
      if (cur_bi >= 0) flush_blocks(blk, cur_bi, A.grid, bj, bj_lo, bj_hi, acc, lane);
    }
    bar_sync(kBarEnd, nthr);
    if (warp == 1) score_frame(A, blk, blkn, wlr, pk, ff, lane);
    bar_sync(kBarEnd, nthr);
  }
  if (warp == 1 && lane == 0) fq_finish(A);
}

// ------------------------------------------------- identity downsample (out == source)
// When the target resolution equals the source (BASELINE configs[0]: 50x50 frames),
// O1 is the identity, so the source frame IS the small frame and the t-k anchor is
// source frame f-k itself (or the state ring before tau0): no band pipeline and no
// cross-CTA anchor hand-off are needed.  One CTA per needed frame (grid-stride):
// 16-byte vectors are copied to the small-frame buffer and, for scored frames, the
// integer SSD against the anchor is accumulated per LR block (per-thread partials,
// u32 smem atomics when the block changes); then the fp64 score in the fixed order
// of O3 and the disposition of O4 — the same arithmetic as dd_kernel.
constexpr int kIdThreads = 256;

__global__ void __launch_bounds__(kIdThreads)
dd_identity_kernel(DsArgs A) {
  __shared__ uint32_t blk[kMaxGrid * kMaxGrid + 2];
  __shared__ uint32_t blkn[kMaxGrid * kMaxGrid + 2];
  __shared__ double wlr[kMaxGrid * kMaxGrid + 2];
  __shared__ double pk[kMaxGrid * kMaxGrid + 2];
  const int tid = threadIdx.x, lane = tid & 31;
  const int gg = A.grid * A.grid;
  const int n_out = A.out_w * 3;
  const int small_bytes = n_out * A.out_h;
  const int nvec = (small_bytes + 15) >> 4;
  if (A.metric == 1) {
    const int sh = A.out_h / A.grid, sw = A.out_w / A.grid;
    for (int q = tid; q < gg; q += blockDim.x) {
      const int bi = q / A.grid, bj = q % A.grid;
      const int rows = bi < A.grid - 1 ? sh : A.out_h - (A.grid - 1) * sh;
      const int cols = bj < A.grid - 1 ? sw : A.out_w - (A.grid - 1) * sw;
      blkn[q] = (uint32_t)(rows * cols * 3);
      wlr[q] = (double)A.lr_w[q];
    }
  }
  for (int q = tid; q < gg; q += blockDim.x) blk[q] = 0u;
  __syncthreads();
  for (int64_t m = A.need.m0 + blockIdx.x; m < A.need.m1; m += gridDim.x) {
    const int64_t f = frame_of(A.need, m);
    const int64_t tau = A.tau0 + f;
    const bool checked = A.t_skip == 1 || (tau % A.t_skip) == 0;
    const bool forced = A.mode == 1 && checked && tau < A.k;
    const bool scoring = checked && !forced;
    const uint8_t* src = A.frames + f * A.frame_pitch;
    uint8_t* dst = A.small + f * A.small_pitch;
    const uint8_t* anc = A.ref;
    if (A.mode == 1 && scoring)
      anc = f - A.k >= 0 ? A.frames + (f - A.k) * A.frame_pitch : A.ring + ((tau - A.k) % A.k) * A.ring_pitch;
    for (int v = tid; v < nvec; v += blockDim.x) {
      const uint4 w = reinterpret_cast<const uint4*>(src)[v];
      reinterpret_cast<uint4*>(dst)[v] = w;  // pitches are 16-byte multiples
      if (!scoring) continue;
      const int x0 = v << 4;
      uint32_t a[4];
      if (x0 + 16 <= small_bytes && (reinterpret_cast<uintptr_t>(anc) & 15) == 0) {
        const uint4 av = *reinterpret_cast<const uint4*>(anc + x0);
        a[0] = av.x; a[1] = av.y; a[2] = av.z; a[3] = av.w;
      } else {  // tail or unaligned reference image: byte loads inside the image only
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t word = 0;
          for (int b = 0; b < 4; ++b)
            if (x0 + 4 * j + b < small_bytes) word |= (uint32_t)anc[x0 + 4 * j + b] << (8 * b);
          a[j] = word;
        }
      }
      const uint32_t s[4] = {w.x, w.y, w.z, w.w};
      int row = x0 / n_out, colb = x0 - row * n_out;  // byte column within the row
      uint32_t acc = 0u;
      int cur = -1;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        if (x0 + e < small_bytes) {
          const int d = (int)((s[e >> 2] >> (8 * (e & 3))) & 0xFFu) - (int)((a[e >> 2] >> (8 * (e & 3))) & 0xFFu);
          const int q = A.metric == 1 ? block_of(row, A.out_h, A.grid) * A.grid + block_of(colb / 3, A.out_w, A.grid) : 0;
          if (q != cur) {
            if (cur >= 0 && acc) atomicAdd(&blk[cur], acc);
            cur = q;
            acc = 0u;
          }
          acc += (uint32_t)(d * d);
        }
        if (++colb == n_out) {
          colb = 0;
          ++row;
        }
      }
      if (cur >= 0 && acc) atomicAdd(&blk[cur], acc);
    }
    __syncthreads();
    if (tid < 32) {
      if (scoring) {
        if (A.metric == 0) {
          if (lane == 0) {
            const double sc = (double)blk[0] / (double)small_bytes;
            blk[0] = 0u;
            A.score[f] = sc;
            A.disp[f] = sc > A.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
          }
        } else {
          for (int q = lane; q < gg; q += 32) {
            pk[q] = __dmul_rn(wlr[q], (double)blk[q] / (double)blkn[q]);  // w_k * m_k, rounded
            blk[q] = 0u;
          }
          __syncwarp();
          if (lane == 0) {
            double z = (double)A.lr_b;
            for (int q = 0; q < gg; ++q) z = __dadd_rn(z, pk[q]);  // fixed order, no FMA
            if (z != z) atomicOr(A.status, 1u);
            A.score[f] = z;
            A.disp[f] = z > A.delta ? NOSCOPE_FIRED : NOSCOPE_SUPPRESSED;
          }
        }
      } else if (forced && lane == 0) {
        A.score[f] = __longlong_as_double(0x7FF0000000000000ll);  // +inf
        A.disp[f] = NOSCOPE_FIRED;
      }
    }
    __syncthreads();
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
    // both pitches are multiples of 16 (16-byte vectors; the tail of the last vector
    // is the pitch padding on both sides)
    const int nv = (small_bytes + 15) / 16;
    for (int t = threadIdx.x; t < nv; t += blockDim.x)
      reinterpret_cast<uint4*>(dst)[t] = reinterpret_cast<const uint4*>(src)[t];
  }
  if (labels && blockIdx.x == 0) {
    const int64_t lf = n - lh > 0 ? n - lh : 0;
    for (int64_t f = lf + threadIdx.x; f < n; f += blockDim.x)
      lab_hist[(tau0 + f) % lh] = labels[f];
  }
}

// ===================================================================== host
// Launch geometry of dd_kernel: band stage size, worker groups (NG) x column
// segments (NS), ring stages per group, per-warp column-sum words, dynamic smem.
static size_t ds_plan(DsArgs& A, int ctas_per_sm) {
  int stage = 0;
  for (int i = 0; i < A.out_h; ++i) {
    const int r0 = (i * A.H) / A.out_h, r1 = ((i + 1) * A.H) / A.out_h;
    const int64_t b0 = (int64_t)r0 * A.RB, b1 = (int64_t)r1 * A.RB;
    const int64_t a0 = b0 & ~15ll, a1 = (b1 + 15) & ~15ll;
    if ((int)(a1 - a0) > stage) stage = (int)(a1 - a0);
  }
  A.stage_bytes = (stage + 127) & ~127;
  // segments of <= 10 output pixels (<= 30 lanes own one output value each)
  A.ns = std::max(1, (A.out_w + 9) / 10);
  int ng_max = 4;  // 4 bands in flight per CTA (A/B on B200: 2 -> 17.3 ms, 3 -> 15.8, 4 -> 15.0, 5 -> 15.2)
  if (const char* e = std::getenv("NOSCOPE_DD_NG")) ng_max = std::atoi(e);
  ng_max = std::max(1, std::min({ng_max, kDsMaxGroups, A.out_h, kDsMaxWorkers / A.ns}));
  int cs = 0;
  for (int g = 0; g < A.ns; ++g) cs = std::max(cs, segment_of(g, A.ns, A.out_w, A.W, A.fast != 0).span);
  A.cs_stride = (cs + 7) & ~7;
  const int gg2 = ((A.grid * A.grid) + 1) & ~1;
  const int small_bytes = A.out_w * A.out_h * 3;
  auto up = [](size_t x, size_t a) { return (x + a - 1) / a * a; };
  const size_t per_cta = (size_t)(227 * 1024) / ctas_per_sm - 1024;  // less the 1 KB per-CTA reservation
  // Fewer worker groups when bands are large (720p / 1080p sources): every group
  // needs a ring of >= 2 stages of one band each.
  size_t b = 0;
  for (int ng = ng_max; ng >= 1; --ng) {
    A.ng = ng;
    b = kDsHeadBytes + (size_t)A.out_h * sizeof(BandInfo);
    A.off_ref = (int)b;
    b += A.mode == 0 ? (size_t)((small_bytes + 15) & ~15) : 0;   // reference image (mode 0)
    A.off_blkn = (int)(b = up(b, 16));
    b += (size_t)gg2 * 4;
    A.off_blk = (int)(b = up(b, 16));
    b += 2 * (size_t)gg2 * 4;                                   // blk[2] (frame parity)
    A.off_wlr = (int)(b = up(b, 16));
    b += 2 * (size_t)gg2 * 8;                                   // wlr, pk
    A.off_cs = (int)(b = up(b, 16));
    b += (size_t)A.ng * A.ns * A.cs_stride * sizeof(uint16_t);
    A.off_stages = (int)(b = up(b, 128));
    // ring: as many stages per group as fit
    int nsg = per_cta > b ? (int)((per_cta - b) / ((size_t)A.ng * A.stage_bytes)) : 0;
    A.nsg = std::min(nsg, kDsMaxStages / A.ng);
    if (A.nsg >= 2) break;
  }
  return b + (size_t)A.ng * A.nsg * A.stage_bytes;
}

bool dd_uses_band_kernel(const noscope_dd_config& cfg, const noscope_frames_desc& desc) {
  const int grid = cfg.metric == 1 ? cfg.grid : 1;
  return !(desc.width == cfg.out_w && desc.height == cfg.out_h && grid <= kMaxGrid);
}

bool dd_frames_fit(const noscope_dd_config& cfg, const noscope_frames_desc& desc) {
  if (desc.width == cfg.out_w && desc.height == cfg.out_h) return true;   // identity kernel, no bands
  DsArgs A{};
  A.W = desc.width;
  A.H = desc.height;
  A.RB = desc.width * 3;
  A.out_w = cfg.out_w;
  A.out_h = cfg.out_h;
  A.mode = cfg.mode;
  A.grid = cfg.metric == 1 ? cfg.grid : 1;
  A.fast = (A.RB % 16) == 0;
  ds_plan(A, 1);
  return A.nsg >= 2;
}

size_t dd_flags_bytes() { return (size_t)4 * kNumSMs * 4; }

noscope_status launch_diff_detect(const noscope_dd_config& cfg, const uint8_t* frames,
                                  const noscope_frames_desc& desc, int64_t n, int64_t tau0,
                                  uint8_t* state, uint8_t* small, int64_t small_pitch,
                                  double* score, uint8_t* disp, uint32_t* status, unsigned* flags,
                                  cudaStream_t st, Prof* prof, FiredQueue* fq, int reserve_sms) {
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
  // per-block / per-frame SSDs are u32 (255^2 per output value)
  if ((int64_t)A.out_w * A.out_h * 3 * 65025 >= ((int64_t)1 << 32)) return NOSCOPE_SHAPE;
  int cps = 1;  // CTAs per SM (timing experiments: NOSCOPE_DD_CPS)
  if (const char* e = std::getenv("NOSCOPE_DD_CPS")) cps = std::max(1, std::min(4, std::atoi(e)));
  size_t smem = ds_plan(A, cps);
  while (A.nsg < 2 && cps > 1) smem = ds_plan(A, --cps);
  if (A.nsg < 2) return NOSCOPE_SHAPE;
  const int threads = (2 + A.ng * A.ns) * 32;
  // compile-time geometry for the 640x480 -> 50x50 webcam stream (bands of 9/10 rows,
  // boxes of 12/13 pixels, 1,920-byte rows); everything else takes the generic kernel
  void (*kern)(DsArgs) = dd_kernel<0, 0, 0>;
  if (A.fast && A.rlo == 9 && A.W / A.out_w == 12 && A.RB == 1920) kern = dd_kernel<9, 12, 120>;
  const int64_t frames_needed = A.need.m1 - A.need.m0;
  if (A.W == A.out_w && A.H == A.out_h && A.grid <= kMaxGrid) {  // O1 is the identity
    if (fq) return NOSCOPE_INVALID_ARGUMENT;   // no fired-frame queue on this path
    if (frames_needed > 0) {
      const int grid = (int)std::min<int64_t>(frames_needed, (int64_t)kNumSMs * 8);
      dd_identity_kernel<<<grid, kIdThreads, 0, st>>>(A);
      NS_LAUNCH_CHECK();
      count_launch();
    }
    prof_mark(prof, st);
    return NOSCOPE_OK;
  }
  if (frames_needed > 0) {
    static DeviceOnce attr_set[2];
    const int ki = kern == dd_kernel<0, 0, 0> ? 0 : 1;
    if (attr_set[ki].first())
      NS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    int per_sm = 0;
    NS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    if (per_sm < 1) return NOSCOPE_SHAPE;
    int sms = kNumSMs, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (const char* e = std::getenv("NOSCOPE_DD_SMS")) sms = std::max(1, std::min(sms, std::atoi(e)));  // experiments
    sms = std::max(1, sms - std::max(0, reserve_sms));
    // all CTAs co-resident (deferred scoring waits on earlier CTAs' flags)
    const int grid = (int)std::min<int64_t>(frames_needed, (int64_t)std::min(per_sm, cps) * sms);
    if (fq) {
      fq->producers = grid;
      A.fq = *fq;
    }
    if (cfg.mode == 1) NS_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)grid * 4, st));
    NS_CUDA_TRY(launch_cooperative(kern, grid, threads, smem, st, A));  // deferred anchors wait on earlier CTAs
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
