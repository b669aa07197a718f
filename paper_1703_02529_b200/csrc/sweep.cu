// sweep.cu — the CBO's (delta_diff, c_low, c_high) threshold sweep
// (§6.3, cost model P:685-701, objective P:627-637).
//
// The paper sorts frames by the DD metric and sweeps prefixes; here the same
// exact counts come from a histogram over candidate bins, which is what makes
// the sweep a bandwidth-bound pass over the labelled records and lets GPUs
// sum partial histograms (NCCL allreduce between phase 1 and phase 2):
//   d = #{j : delta_j < s}       (frame fired for exactly the j < d)
//   b = #{u < z} + #{u <= z}     (c_lt = b/2 floor, c_le = b/2 ceil)
//   H2[d][b][y] += 1,  H1[d][a][y] += 1
// Phase 2 turns suffix sums over d and prefix/suffix sums over b into the
// per-threshold tables FP/FN/F/U and evaluates all n_delta*m*(m+1)/2 triples
// with the integer cost model, reducing to the lexicographic argmin.
#include "common.cuh"
#include "internal.h"

namespace ns {

// 1,024 threads x 4 records in flight per thread (1e9 records: 6.41 ms; 512 x 8: 7.59,
// 1,024 x 2 / 5 / 6 / 8: 6.51 / 6.43 / 7.31 / 9.08, 768 x 4: 6.67, 512 x 16: 15.15);
// with the vector record loads 5.91 ms (1,024 x 8: 7.08, 512 x 8: 6.41, 512 x 4: 6.82;
// NS_HIST_T / NS_HIST_U override for such A/Bs, tools/gpu_hist_shape.sh)
#ifndef NS_HIST_T
#define NS_HIST_T 1024
#endif
#ifndef NS_HIST_U
#define NS_HIST_U 4
#endif
constexpr int kHistThreads = NS_HIST_T;
constexpr int kHistU = NS_HIST_U;
constexpr int kMaxCand = 2048;

struct HistLayout {
  int nd, m, B;         // B = 2m + 1
  size_t h2, h1, tail;  // word offsets
  size_t words;
  __host__ __device__ HistLayout(int nd_, int m_) : nd(nd_), m(m_), B(2 * m_ + 1) {
    h2 = 0;
    h1 = (size_t)(nd + 1) * B * 2;
    tail = h1 + (size_t)(nd + 1) * 4;
    words = tail + 2;
  }
};

// Smallest power of two P with P >= n + 1 (so a P-step search can return n).
__host__ __device__ inline int pow2_above(int n) {
  int p = 1;
  while (p < n + 1) p <<= 1;
  return p;
}

NS_DEV int count_lt_d(const double* c, int n, double v) {  // #{c < v}
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (c[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
NS_DEV int count_lt_f(const float* c, int n, float v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (c[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
NS_DEV int count_le_f(const float* c, int n, float v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (c[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// The candidate searches walk an implicit binary tree stored in BFS (Eytzinger)
// order: node k's children are 2k+1 and 2k+2, so one level's nodes are
// contiguous (the top levels are conflict-free broadcasts; on the sorted array
// the pivots of one level sit a power of two apart, all in one bank: ~34
// wavefronts per warp for a 128-entry f64 search) and a step is one load, one
// compare and one IMAD: k = 2k + 1 + (tree[k] < x).  With P = 2^h leaves the
// tree holds the P - 1 sorted candidates (+inf padded) and, after h steps,
// k - (P - 1) = #{candidates < x}.
// In-order (sorted) index of BFS node i of the perfect tree with 2^h - 1 nodes.
NS_DEV int eytz_sorted_index(int i, int h) {
  const int d = 31 - __clz(i + 1);            // depth
  const int p = i + 1 - (1 << d);             // position in its level
  return ((2 * p + 1) << (h - 1 - d)) - 1;
}

// Phase 1: block-privatised histogram in shared memory (u32), flushed to the
// global u64 histogram with one atomic per nonzero bin.  HD / HU: the search depths
// fixed at compile time (fully unrolled searches; the kernel is issue-bound), 0 = the
// runtime depths.
template <int HD, int HU>
__global__ void __launch_bounds__(kHistThreads, 1)
sweep_hist_kernel(const double* __restrict__ s, const float* __restrict__ z,
                  const uint8_t* __restrict__ y, const uint8_t* __restrict__ a, int64_t n,
                  const double* __restrict__ delta, int nd, const float* __restrict__ u, int m,
                  unsigned long long* hist, uint32_t* status, int privatised) {
  extern __shared__ __align__(16) uint8_t smem[];
  HistLayout L(nd, m);
  const int pd = pow2_above(nd), pu = pow2_above(m);
  const int hd = HD ? HD : 31 - __clz(pd), hu = HU ? HU : 31 - __clz(pu);
  double* dt = reinterpret_cast<double*>(smem);            // [pd] BFS tree of the delta candidates
  float* ut = reinterpret_cast<float*>(dt + pd);            // [pu] BFS tree of the logit candidates
  float* uc = ut + pu;                                      // [pu] sorted logit candidates (equality test)
  uint32_t* hs = reinterpret_cast<uint32_t*>(uc + pu);
  const int tid = threadIdx.x;
  const double dinf = __longlong_as_double(0x7FF0000000000000ll);
  const float finf = __int_as_float(0x7F800000);
  for (int t = tid; t < pd - 1; t += blockDim.x) {
    const int q = eytz_sorted_index(t, hd);
    dt[t] = q < nd ? delta[q] : dinf;
  }
  for (int t = tid; t < pu - 1; t += blockDim.x) {
    const int q = eytz_sorted_index(t, hu);
    ut[t] = q < m ? u[q] : finf;
  }
  for (int t = tid; t < pu; t += blockDim.x) uc[t] = t < m ? u[t] : finf;
  if (privatised)
    for (size_t t = tid; t < L.tail; t += blockDim.x) hs[t] = 0u;
  __syncthreads();
  unsigned long long checked = 0;
  bool bad = false;
  const uint32_t h2o = (uint32_t)L.h2, h1o = (uint32_t)L.h1;
  const double ninf = __longlong_as_double(0xFFF0000000000000ll);
  // Each thread takes kU records per step (all loads issued before the searches,
  // record = chunk base + tid * kU + r), so the dependent
  // binary-search chains of independent records overlap.
  // The next step's records are prefetched into registers before the current
  // step's searches run (software pipelining: loads overlap the search work).
  constexpr int kU = kHistU;
  const int64_t step = (int64_t)gridDim.x * blockDim.x * kU;
  double sv[kU], sn[kU];
  float zv[kU], zn[kU];
  uint32_t ya[kU], yn[kU];
  // kU consecutive records per thread: with aligned columns, one 16-byte load per
  // two s / four z and one 4-byte load of y and of a (a warp still reads contiguous
  // runs); unaligned columns or the ragged end fall back to per-record loads.
  const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(z)) & 15) == 0 &&
                   ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(a)) & 3) == 0;
  static_assert(kHistU % 4 == 0, "vector record loads take records in fours");
  auto load = [&](int64_t base, double (&sx)[kU], float (&zx)[kU], uint32_t (&yx)[kU]) {
    const int64_t i0 = base + (int64_t)tid * kU;
    if (vec && i0 + kU <= n) {
#pragma unroll
      for (int q = 0; q < kU / 4; ++q) {
        const double2 s01 = __ldcs(reinterpret_cast<const double2*>(s + i0 + 4 * q));
        const double2 s23 = __ldcs(reinterpret_cast<const double2*>(s + i0 + 4 * q + 2));
        const float4 z4 = __ldcs(reinterpret_cast<const float4*>(z + i0 + 4 * q));
        const uint32_t y4 = __ldcs(reinterpret_cast<const unsigned int*>(y + i0 + 4 * q));
        const uint32_t a4 = __ldcs(reinterpret_cast<const unsigned int*>(a + i0 + 4 * q));
        sx[4 * q] = s01.x; sx[4 * q + 1] = s01.y; sx[4 * q + 2] = s23.x; sx[4 * q + 3] = s23.y;
        zx[4 * q] = z4.x; zx[4 * q + 1] = z4.y; zx[4 * q + 2] = z4.z; zx[4 * q + 3] = z4.w;
#pragma unroll
        for (int r = 0; r < 4; ++r)
          yx[4 * q + r] = ((y4 >> (8 * r)) & 0xFFu) | (((a4 >> (8 * r)) & 0xFFu) << 8);
      }
      return;
    }
#pragma unroll
    for (int r = 0; r < kU; ++r) {
      const int64_t i = i0 + r;
      if (i < n) {
        sx[r] = __ldcs(s + i);
        zx[r] = __ldcs(z + i);
        yx[r] = (uint32_t)__ldcs(y + i) | ((uint32_t)__ldcs(a + i) << 8);
      } else {
        sx[r] = 0.0;
        zx[r] = 0.0f;
        yx[r] = 0x10000u;  // no record
      }
    }
  };
  int64_t base = (int64_t)blockIdx.x * blockDim.x * kU;
  if (base < n) load(base, sn, zn, yn);
  for (; base < n; base += step) {
#pragma unroll
    for (int r = 0; r < kU; ++r) {
      sv[r] = sn[r];
      zv[r] = zn[r];
      ya[r] = yn[r];
    }
    if (base + step < n) load(base + step, sn, zn, yn);
    // Branch-free binary searches over the +inf-padded power-of-two grids, all
    // 2*kU searches advanced one level at a time (independent smem chains).
    int dj[kU], lj[kU];
#pragma unroll
    for (int r = 0; r < kU; ++r) dj[r] = lj[r] = 0;
    for (int lv = 0; lv < hd; ++lv) {   // constant trip count (fully unrolled) when HD != 0
#pragma unroll
      for (int r = 0; r < kU; ++r) dj[r] = 2 * dj[r] + 1 + (dt[dj[r]] < sv[r] ? 1 : 0);
    }
    for (int lv = 0; lv < hu; ++lv) {
#pragma unroll
      for (int r = 0; r < kU; ++r) lj[r] = 2 * lj[r] + 1 + (ut[lj[r]] < zv[r] ? 1 : 0);
    }
#pragma unroll
    for (int r = 0; r < kU; ++r) {
      dj[r] -= pd - 1;    // #{delta < s}
      lj[r] -= pu - 1;    // #{u < z}
    }
#pragma unroll
    for (int r = 0; r < kU; ++r) {
      if (ya[r] & 0x10000u) continue;
      const double si = sv[r];
      const float zi = zv[r];
      const int yi = (ya[r] & 0xFFu) ? 1 : 0, ai = (ya[r] & 0xFF00u) ? 1 : 0;
      bad |= (si != si) | (zi != zi);
      checked += (si != ninf);
      const int d = dj[r];
      const int lt = lj[r];
      const int b = 2 * lt + ((lt < m && uc[lt] == zi) ? 1 : 0);  // #{u<z} + #{u<=z}
      // 32-bit word indices: the histogram has < 2^30 words (nd < 65536, m <= 2048)
      const uint32_t w2 = h2o + ((uint32_t)d * (uint32_t)L.B + (uint32_t)b) * 2u + (uint32_t)yi;
      const uint32_t w1 = h1o + (uint32_t)d * 4u + (uint32_t)(ai * 2 + yi);
      // H1 is only ever read at (a, y) = (1, 0) and (0, 1) (the not-fired FP and
      // FN counts), so records with a == y skip that atomic (shared-memory
      // atomics are this kernel's throughput limit).
      const bool h1 = ai != yi;
      if (privatised) {
        atomicAdd(&hs[w2], 1u);
        if (h1) atomicAdd(&hs[w1], 1u);
      } else {
        atomicAdd(&hist[w2], 1ull);
        if (h1) atomicAdd(&hist[w1], 1ull);
      }
    }
  }
  if (bad) atomicOr(status, 4u);
  checked = warp_sum(checked);
  if ((tid & 31) == 0 && checked) atomicAdd(&hist[L.tail], checked);
  if (privatised) {
    __syncthreads();
    for (size_t t = tid; t < L.tail; t += blockDim.x)
      if (hs[t]) atomicAdd(&hist[t], (unsigned long long)hs[t]);
  }
  if (blockIdx.x == 0 && tid == 0) atomicAdd(&hist[L.tail + 1], (unsigned long long)n);
}

// Phase 2a: per-delta tables.
// sweep_dsuffix_kernel: one warp per histogram column, one pass over d —
//   G[d][b][y] = sum_{d' >= d} H2[d'][b][y]   (fired under delta_j  <=>  d > j)
//   Pn[d][c]   = sum_{d' <= d} H1[d'][c]      (c = (a=1,y=0), (a=0,y=1); not fired <=> d <= j)
struct Tables {
  unsigned long long *F, *FPnf, *FNnf, *FPf, *FNf, *GE, *GT;
};

__global__ void sweep_dsuffix_kernel(const unsigned long long* __restrict__ hist, int nd, int m,
                                     unsigned long long* __restrict__ G, unsigned long long* __restrict__ Pn) {
  // one warp per column; the d axis in slices of 32 (lane = d), scanned with shuffles
  HistLayout L(nd, m);
  const int cols = 2 * L.B;
  const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (c < cols) {
    unsigned long long carry = 0;   // sum over the d already done (above this slice)
    for (int top = nd; top >= 0; top -= 32) {
      const int d = top - lane;     // lane 0 = largest d of the slice
      unsigned long long v = d >= 0 ? hist[L.h2 + (size_t)d * cols + c] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {      // inclusive scan towards smaller d
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (d >= 0) G[(size_t)d * cols + c] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  } else if (c < cols + 2) {
    const int w = c == cols ? 1 * 2 + 0 : 0 * 2 + 1;   // (a, y) = (1, 0) FP, (0, 1) FN
    unsigned long long carry = 0;
    for (int d0 = 0; d0 <= nd; d0 += 32) {
      const int d = d0 + lane;
      unsigned long long v = d <= nd ? hist[L.h1 + (size_t)d * 4 + w] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (d <= nd) Pn[(size_t)d * 2 + (c - cols)] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
}

// One CTA per j: the fired histogram over logit bins (G at d = j + 1), then
// suffix / prefix sums over b.
__global__ void sweep_prefix_kernel(const unsigned long long* __restrict__ G,
                                    const unsigned long long* __restrict__ Pn, int nd, int m, Tables T) {
  extern __shared__ __align__(16) uint8_t smem[];
  HistLayout L(nd, m);
  unsigned long long* fh0 = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* fh1 = fh0 + L.B;
  unsigned long long* S0 = fh1 + L.B;   // suffix of fh0
  unsigned long long* SA = S0 + L.B + 1;  // suffix of fh0 + fh1
  unsigned long long* P1 = SA + L.B + 1;  // prefix (inclusive) of fh1
  const int j = blockIdx.x, tid = threadIdx.x;
  const unsigned long long* g = G + (size_t)(j + 1) * 2 * L.B;
  for (int b = tid; b < L.B; b += blockDim.x) {
    fh0[b] = g[2 * b + 0];
    fh1[b] = g[2 * b + 1];
  }
  __syncthreads();
  // suffix sums of fh0 and fh0 + fh1 and the prefix sum of fh1 over b, by warp 0:
  // 32 lanes per slice with shuffle scans, a carry between slices (B <= 4097)
  if (tid < 32) {
    const int lane = tid;
    unsigned long long c0 = 0, cA = 0;
    for (int top = L.B - 1; top >= 0; top -= 32) {
      const int b = top - lane;
      unsigned long long v0 = b >= 0 ? fh0[b] : 0ull, vA = b >= 0 ? fh0[b] + fh1[b] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y0 = __shfl_up_sync(0xffffffffu, v0, o);
        const unsigned long long yA = __shfl_up_sync(0xffffffffu, vA, o);
        if (lane >= o) {
          v0 += y0;
          vA += yA;
        }
      }
      if (b >= 0) {
        S0[b] = c0 + v0;
        SA[b] = cA + vA;
      }
      c0 += __shfl_sync(0xffffffffu, v0, 31);
      cA += __shfl_sync(0xffffffffu, vA, 31);
    }
    unsigned long long c1 = 0;
    for (int b0 = 0; b0 < L.B; b0 += 32) {
      const int b = b0 + lane;
      unsigned long long v1 = b < L.B ? fh1[b] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y1 = __shfl_up_sync(0xffffffffu, v1, o);
        if (lane >= o) v1 += y1;
      }
      if (b < L.B) P1[b] = c1 + v1;
      c1 += __shfl_sync(0xffffffffu, v1, 31);
    }
    __syncwarp();   // SA[0] was written by another lane
    if (lane == 0) {
      S0[L.B] = 0;
      SA[L.B] = 0;
      T.F[j] = SA[0];
      T.FPnf[j] = Pn[(size_t)j * 2 + 0];
      T.FNnf[j] = Pn[(size_t)j * 2 + 1];
    }
  }
  __syncthreads();
  for (int t = tid; t < m; t += blockDim.x) {
    const int bg = 2 * t + 2 < L.B ? 2 * t + 2 : L.B;   // z > u_t  <=> b >= 2t+2
    const int be = 2 * t + 1;                           // z >= u_t <=> b >= 2t+1
    T.FPf[(size_t)j * m + t] = S0[bg];
    T.GT[(size_t)j * m + t] = SA[bg];
    T.GE[(size_t)j * m + t] = SA[be];
    T.FNf[(size_t)j * m + t] = P1[2 * t];               // z < u_t  <=> b <= 2t
  }
}

// Phase 2b: evaluate every (j, l <= h).
// Phase-2 work split: the (l, h >= l) triangle of one delta row is cut into
// (m + 1) / 2 row pairs {l, m - 1 - l} of m + 1 cells each (one pair of m - l cells
// when m is odd), dealt round-robin over eval_pieces(m) threads (interleaved, so a
// warp reads consecutive h: strided pieces would put every lane on one bank).
__host__ __device__ inline int eval_pieces(int m) {
  const int p = (m + 1) / 32;
  return p < 1 ? 1 : (p > 32 ? 32 : p);
}
// CTAs per delta row: about 512 cells per thread (each CTA stages the row's FPf and
// GT columns, so more CTAs per row cost more staging than they save).
__host__ __device__ inline int eval_ctas_per_row(int m) {
  const int64_t cells = (int64_t)m * (m + 1) / 2;
  const int64_t c = (cells + 256 * 512 - 1) / (256 * 512);
  return (int)(c < 1 ? 1 : (c > 64 ? 64 : c));
}

struct Cand {
  unsigned long long k0, k1, k2;
  unsigned int j, nl, h, valid;
};
NS_DEV bool cand_less(const Cand& x, const Cand& y) {
  if (x.valid != y.valid) return x.valid > y.valid;
  if (x.k0 != y.k0) return x.k0 < y.k0;
  if (x.k1 != y.k1) return x.k1 < y.k1;
  if (x.k2 != y.k2) return x.k2 < y.k2;
  if (x.j != y.j) return x.j < y.j;
  if (x.nl != y.nl) return x.nl < y.nl;
  return x.h < y.h;
}

// One (j, l, h) cell of the sweep: cost and constraint keys, kept if it beats the
// thread's best feasible (bf) or least-violating (bi) candidate.
NS_DEV void eval_cell(int j, int m, int l, int h, unsigned long long fn, unsigned long long ge,
                      unsigned long long fp, unsigned long long gth, unsigned long long base_cost,
                      unsigned long long t_full, unsigned long long fp_lim, unsigned long long fn_lim,
                      Cand& bf, Cand& bi) {
  const unsigned long long U = ge - gth;
  const unsigned long long cost = base_cost + U * t_full;
  Cand c;
  c.j = j;
  c.nl = (unsigned)(m - 1 - l);
  c.h = h;
  c.valid = 1;
  if (fp <= fp_lim && fn <= fn_lim) {
    c.k0 = cost; c.k1 = U; c.k2 = 0;
    if (cand_less(c, bf)) bf = c;
  } else {
    const unsigned long long vfp = fp > fp_lim ? fp - fp_lim : 0;
    const unsigned long long vfn = fn > fn_lim ? fn - fn_lim : 0;
    c.k0 = vfp > vfn ? vfp : vfn; c.k1 = cost; c.k2 = U;
    if (cand_less(c, bi)) bi = c;
  }
}

struct EvalOut {
  Cand feas, infeas;
};

// eval_ctas_per_row(m) CTAs per delta row j: the j row of FPf and GT (m entries
// each) staged in shared memory; the CTAs' threads stride over the row's (pair,
// piece) items, the pair's FN and GE entries in registers.
__global__ void __launch_bounds__(256)
sweep_eval_kernel(Tables T, const unsigned long long* hist, int nd, int m,
                  unsigned long long t_mse, unsigned long long t_snn,
                  unsigned long long t_full, unsigned long long fp_lim,
                  unsigned long long fn_lim, EvalOut* block_out) {
  extern __shared__ __align__(16) uint8_t esm[];
  unsigned long long* fpf = reinterpret_cast<unsigned long long*>(esm);   // [m]
  unsigned long long* gt = fpf + m;                                        // [m]
  __shared__ Cand sf[256], si[256];
  HistLayout L(nd, m);
  const int cpr = eval_ctas_per_row(m), P = eval_pieces(m);
  const int j = blockIdx.x / cpr;
  for (int h = threadIdx.x; h < m; h += blockDim.x) {
    fpf[h] = T.FPf[(size_t)j * m + h];
    gt[h] = T.GT[(size_t)j * m + h];
  }
  __syncthreads();
  Cand bf{0, 0, 0, 0, 0, 0, 0}, bi{0, 0, 0, 0, 0, 0, 0};
  const unsigned long long checked = hist[L.tail];
  const unsigned long long F = T.F[j];
  const unsigned long long fpnf = T.FPnf[j], fnnf = T.FNnf[j];
  const unsigned long long base_cost = checked * t_mse + F * t_snn;
  const unsigned long long* fnf = T.FNf + (size_t)j * m;
  const unsigned long long* ger = T.GE + (size_t)j * m;
  const int items = ((m + 1) / 2) * P;   // (pair, piece) work items of this row
  for (int w = (blockIdx.x - j * cpr) * blockDim.x + threadIdx.x; w < items; w += cpr * blockDim.x) {
    const int r = w / P, p = w - r * P;
    const int l1 = r, l2 = m - 1 - r;
    const int len1 = m - l1, tot = l2 > l1 ? m + 1 : len1;
    const unsigned long long fn1 = fnnf + fnf[l1], ge1 = ger[l1];
    const unsigned long long fn2 = fnnf + fnf[l2], ge2 = ger[l2];
    // lanes on consecutive cells (conflict-free smem reads); the pair's two rows as
    // two loops, so the cell body carries no per-cell row select
    int i = p;
    for (; i < len1; i += P)
      eval_cell(j, m, l1, l1 + i, fn1, ge1, fpnf + fpf[l1 + i], gt[l1 + i], base_cost, t_full, fp_lim,
                fn_lim, bf, bi);
    for (; i < tot; i += P)
      eval_cell(j, m, l2, l2 + (i - len1), fn2, ge2, fpnf + fpf[l2 + (i - len1)], gt[l2 + (i - len1)],
                base_cost, t_full, fp_lim, fn_lim, bf, bi);
  }
  sf[threadIdx.x] = bf;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      if (cand_less(sf[threadIdx.x + o], sf[threadIdx.x])) sf[threadIdx.x] = sf[threadIdx.x + o];
      if (cand_less(si[threadIdx.x + o], si[threadIdx.x])) si[threadIdx.x] = si[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    block_out[blockIdx.x].feas = sf[0];
    block_out[blockIdx.x].infeas = si[0];
  }
}

__global__ void sweep_final_kernel(const EvalOut* blocks, int nblocks, Tables T,
                                   const unsigned long long* hist, int nd, int m,
                                   const double* delta, const float* u,
                                   unsigned long long t_mse, unsigned long long t_snn,
                                   unsigned long long t_full, noscope_sweep_best* out) {
  // 256 threads stride over the block results, then a shared-memory tree (the
  // key order is total, so the reduction order does not change the result)
  __shared__ Cand sf[256], si[256];
  HistLayout L(nd, m);
  Cand bf{0, 0, 0, 0, 0, 0, 0}, bi{0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
    if (cand_less(blocks[b].feas, bf)) bf = blocks[b].feas;
    if (cand_less(blocks[b].infeas, bi)) bi = blocks[b].infeas;
  }
  sf[threadIdx.x] = bf;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      if (cand_less(sf[threadIdx.x + o], sf[threadIdx.x])) sf[threadIdx.x] = sf[threadIdx.x + o];
      if (cand_less(si[threadIdx.x + o], si[threadIdx.x])) si[threadIdx.x] = si[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  bf = sf[0];
  bi = si[0];
  const bool feasible = bf.valid != 0;
  const Cand c = feasible ? bf : bi;
  noscope_sweep_best r{};
  r.j = (int)c.j;
  r.l = m - 1 - (int)c.nl;
  r.h = (int)c.h;
  r.feasible = feasible ? 1 : 0;
  const unsigned long long F = T.F[r.j];
  r.fp = T.FPnf[r.j] + T.FPf[(size_t)r.j * m + r.h];
  r.fn = T.FNnf[r.j] + T.FNf[(size_t)r.j * m + r.l];
  r.uncertain = T.GE[(size_t)r.j * m + r.l] - T.GT[(size_t)r.j * m + r.h];
  r.fired = F;
  r.checked = hist[L.tail];
  r.total = hist[L.tail + 1];
  r.cost_ps = r.checked * t_mse + F * t_snn + r.uncertain * t_full;
  r.delta = delta[r.j];
  r.lo_logit = u[r.l];
  r.hi_logit = u[r.h];
  *out = r;
}

// ===================================================================== host
size_t sweep_ws_bytes(int32_t nd, int32_t m) {
  size_t tabs = (size_t)nd * 3 + (size_t)nd * m * 4;
  size_t suffix = (size_t)(nd + 1) * (2 * (2 * (size_t)m + 1)) + (size_t)(nd + 1) * 2;
  size_t blocks = (size_t)nd * eval_ctas_per_row(m);
  return 256 + (tabs + suffix) * 8 + blocks * sizeof(EvalOut) + sizeof(noscope_sweep_best) + 256;
}

noscope_status launch_sweep(int32_t phase, const double* s, const float* z, const uint8_t* y,
                            const uint8_t* a, int64_t n, const double* delta, int32_t nd,
                            const float* u, int32_t m, uint64_t* hist_u, const noscope_timing& tm,
                            uint64_t fp_limit, uint64_t fn_limit,
                            const noscope_sweep_tables* tables, noscope_sweep_best* best_host,
                            void* ws, cudaStream_t st, bool* infeasible) {
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(hist_u);
  uint32_t* status = reinterpret_cast<uint32_t*>(ws);
  HistLayout L(nd, m);
  if (phase & 1) {
    if (n > 0) {
      size_t smem = (size_t)pow2_above(nd) * 8 + (size_t)pow2_above(m) * 8;
      size_t priv = smem + L.tail * 4;
      int privatised = priv <= 200 * 1024 ? 1 : 0;
      size_t use = privatised ? priv : smem;
      // set on every call: function attributes are per device context
      // equal search depths 3..11 (8-2047 candidates on both axes; the bench's and
      // configs[3]'s 100-candidate grids: 7) get a fully unrolled instantiation
      const int hd = 31 - __builtin_clz(pow2_above(nd)), hu = 31 - __builtin_clz(pow2_above(m));
      decltype(&sweep_hist_kernel<0, 0>) kern = sweep_hist_kernel<0, 0>;
      switch (hd == hu ? hd : 0) {
        case 3: kern = sweep_hist_kernel<3, 3>; break;
        case 4: kern = sweep_hist_kernel<4, 4>; break;
        case 5: kern = sweep_hist_kernel<5, 5>; break;
        case 6: kern = sweep_hist_kernel<6, 6>; break;
        case 7: kern = sweep_hist_kernel<7, 7>; break;
        case 8: kern = sweep_hist_kernel<8, 8>; break;
        case 9: kern = sweep_hist_kernel<9, 9>; break;
        case 10: kern = sweep_hist_kernel<10, 10>; break;
        case 11: kern = sweep_hist_kernel<11, 11>; break;
        default: break;
      }
      NS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)use));
      int64_t want = (n + kHistThreads * 16 - 1) / (kHistThreads * 16);
      int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, kNumSMs));
      kern<<<grid, kHistThreads, use, st>>>(s, z, y, a, n, delta, nd, u, m, hist, status, privatised);
      NS_LAUNCH_CHECK();
      count_launch();
    }
  }
  if (phase & 2) {
    uint8_t* p = reinterpret_cast<uint8_t*>(ws) + 256;
    Tables T;
    auto take = [&](size_t words) {
      unsigned long long* r = reinterpret_cast<unsigned long long*>(p);
      p += words * 8;
      return r;
    };
    if (tables && tables->F) {
      T.F = reinterpret_cast<unsigned long long*>(tables->F);
      T.FPnf = reinterpret_cast<unsigned long long*>(tables->FPnf);
      T.FNnf = reinterpret_cast<unsigned long long*>(tables->FNnf);
      T.FPf = reinterpret_cast<unsigned long long*>(tables->FPf);
      T.FNf = reinterpret_cast<unsigned long long*>(tables->FNf);
      T.GE = reinterpret_cast<unsigned long long*>(tables->GE);
      T.GT = reinterpret_cast<unsigned long long*>(tables->GT);
      take((size_t)nd * 3 + (size_t)nd * m * 4);
    } else {
      T.F = take(nd);
      T.FPnf = take(nd);
      T.FNnf = take(nd);
      T.FPf = take((size_t)nd * m);
      T.FNf = take((size_t)nd * m);
      T.GE = take((size_t)nd * m);
      T.GT = take((size_t)nd * m);
    }
    unsigned long long* G = take((size_t)(nd + 1) * 2 * L.B);
    unsigned long long* Pn = take((size_t)(nd + 1) * 2);
    const int nblocks = nd * eval_ctas_per_row(m);
    EvalOut* bo = reinterpret_cast<EvalOut*>(p);
    p += (size_t)nblocks * sizeof(EvalOut);
    p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    noscope_sweep_best* best_dev = reinterpret_cast<noscope_sweep_best*>(p);
    const int cols = 2 * L.B + 2;
    sweep_dsuffix_kernel<<<(cols * 32 + 255) / 256, 256, 0, st>>>(hist, nd, m, G, Pn);
    NS_LAUNCH_CHECK();
    const size_t smem = (size_t)(5 * L.B + 2) * 8;   // up to 164 KB at m = 2048
    NS_CUDA_TRY(cudaFuncSetAttribute(sweep_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    sweep_prefix_kernel<<<nd, 256, smem, st>>>(G, Pn, nd, m, T);
    NS_LAUNCH_CHECK();
    count_launch(4);
    NS_CUDA_TRY(cudaFuncSetAttribute(sweep_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)((size_t)m * 16)));
    sweep_eval_kernel<<<nblocks, 256, (size_t)m * 16, st>>>(T, hist, nd, m, tm.t_mse_ps, tm.t_snn_ps,
                                                             tm.t_full_ps, fp_limit, fn_limit, bo);
    NS_LAUNCH_CHECK();
    sweep_final_kernel<<<1, 256, 0, st>>>(bo, nblocks, T, hist, nd, m, delta, u, tm.t_mse_ps,
                                         tm.t_snn_ps, tm.t_full_ps, best_dev);
    NS_LAUNCH_CHECK();
    if (best_host) {
      NS_CUDA_TRY(cudaMemcpyAsync(best_host, best_dev, sizeof(noscope_sweep_best),
                                  cudaMemcpyDeviceToHost, st));
      if (infeasible) {   // synchronous form: the caller gets the result and the status now
        NS_CUDA_TRY(cudaStreamSynchronize(st));
        *infeasible = best_host->feasible == 0;
      }
    }
  }
  return NOSCOPE_OK;
}

}  // namespace ns
