// cnn_gemm.cu — one 3x3 conv + bias + ReLU + 2x2 max-pool layer of the
// specialized CNN (§4: "convolutional layers ... max
// pooling ... the number of filters doubles") as a batched implicit GEMM on
// tcgen05 tensor cores.  Used for every layer that is not inside the fused
// conv1+conv2 kernel (cnn_fused.cu): conv1/conv2 of base_filters = 64 and
// conv3/conv4 of the 4-layer networks.
//
// Data layout: the "stacked" map (internal.h) puts all frames of a chunk one
// after another in one row space with a shared zero separator row/column, so a
// tap (ky, kx) of the 3x3 conv is a constant row shift (ky-1)*Wq + (kx-1) for
// every output row of every frame.  An M tile is 128 consecutive rows of that
// space (spanning frame boundaries freely); its A operand for K step (tap,
// channel-group pair) is a descriptor whose start address is shifted by the
// tap — the 9 taps re-read the same shared-memory block, nothing is expanded.
// Rows that fall on separators are computed and discarded (Wq*(H+1)/(W*H)
// overhead: 8% at 25x25, 17% at 12x12, 36% at 6x6).
//
// Work unit = 128*MT consecutive rows; unit u owns the pool windows whose
// top-left row lies in [c0, c0 + S), S = 128*MT - Wq - 1, so all four rows of
// an owned window are inside the unit (neighbouring units overlap by Wq + 1
// rows, recomputed).
//
// Roles (11 warps, persistent, one CTA per SM):
//   W10   A producer  — cp.async.bulk of the unit's rows (one copy per channel
//                       group plane), nA-deep
//   W0    B producer  — weight K-step slabs [2][N][8] through a bstages ring
//   W1    MMA issuer  — per pass over Cout: steps x MT tcgen05.mma (M=128, N,
//                       K=16), the MT tiles interleaved on independent
//                       accumulators; owns TMEM
//   W2-W9 epilogue    — TMEM -> +bias -> ReLU -> bf16 -> smem staging (16-channel
//                       slabs, double-buffered) -> 2x2 max of the owned windows
//                       -> next layer's stacked map (separators written as zeros)
//                       or the FC feature tiles
#include "common.cuh"
#include "internal.h"

namespace ns {

namespace gm {
constexpr int kThreads = 11 * 32;
constexpr int kEpi = 256;       // epilogue threads (W2-W9)
constexpr int kMaxWin = 1024;   // owned pool windows per unit (<= S/4 + 2*rows/Wq)
constexpr int kNumBars = 2 + 2 + 8 + 8 + 2 + 2;
}  // namespace gm

static size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool make_convg_geom(int cin_real, int cout, int H, int64_t chunk, ConvGGeom* out) {
  ConvGGeom g{};
  g.cin_real = cin_real;
  g.cin_eff = cin_real < 8 ? 8 : cin_real;
  if (g.cin_eff != 8 && g.cin_eff % 16) return false;
  g.cout = cout;
  g.H = H;
  g.W = H;
  g.N = std::min(cout, 256);
  if (cout % g.N || g.N % 16) return false;
  g.passes = cout / g.N;
  // K16 steps: (tap, channel-group pair); Cin = 8 packs two taps per step
  g.steps = g.cin_eff == 8 ? 5 : 9 * (g.cin_eff / 16);
  if (g.N == 256) { g.MT = 2; g.nacc = 1; }
  else if (g.N == 128) { g.MT = 2; g.nacc = 2; }
  else { g.MT = 4; g.nacc = 512 / (4 * g.N) >= 2 ? 2 : 1; }
  const int Wq = g.W + 1;
  g.S = 128 * g.MT - Wq - 1;
  if (g.S <= 0) return false;
  g.rows_blk = 128 * g.MT + 2 * Wq + 3;   // [c0 - Wq - 1, c0 + 128 MT + Wq + 2)
  g.R = sl_rows(g.H, g.W, chunk, 128 * g.MT + Wq + 8);
  uint32_t tc = 32;
  while ((int)tc < g.nacc * g.MT * g.N) tc <<= 1;
  g.tmem_cols = tc;
  const size_t ablk = (size_t)(g.cin_eff / 8) * g.rows_blk * 16;
  auto layout = [&](int nA, int bst) {
    size_t o = al((size_t)nA * ablk, 1024);
    g.oB = o;
    o = al(o + (size_t)bst * g.N * 32, 128);
    g.oStage = o;
    o += (size_t)2 * 128 * g.MT * 32;
    g.oWin = o;
    o += (size_t)gm::kMaxWin * 8;
    g.oBias = o;
    o += (size_t)cout * 4;
    g.oBar = al(o, 8);
    o = g.oBar + gm::kNumBars * 8 + 16;
    return o + 1024;  // alignment slack
  };
  const size_t kMax = 227 * 1024;
  g.nA = 2;
  g.bstages = 6;
  g.smem = layout(2, 6);
  if (g.smem > kMax) { g.nA = 1; g.smem = layout(1, 6); }
  if (g.smem > kMax) { g.bstages = 4; g.smem = layout(1, 4); }
  if (g.smem > kMax) return false;
  *out = g;
  return true;
}

// w [Cout][3][3][Cin_real] bf16 -> out [passes][steps][2][N][8]
__global__ void pack_convg_kernel(const uint16_t* __restrict__ w, ConvGGeom g,
                                  uint16_t* __restrict__ out) {
  const int64_t total = (int64_t)g.cout * g.steps * 16;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t & 7);
    const int64_t r = t >> 3;
    const int n = (int)(r % g.N);
    const int64_t r2 = r / g.N;
    const int h = (int)(r2 & 1);
    const int64_t r3 = r2 >> 1;
    const int s = (int)(r3 % g.steps), p = (int)(r3 / g.steps);
    const int co = p * g.N + n;
    int tap, ch;
    if (g.cin_eff == 8) {
      tap = 2 * s + h;
      ch = e;
    } else {
      const int cpt = g.cin_eff / 16;
      tap = s / cpt;
      ch = ((s % cpt) * 2 + h) * 8 + e;
    }
    out[t] = (tap < 9 && ch < g.cin_real) ? w[((int64_t)co * 9 + tap) * g.cin_real + ch] : 0;
  }
}

noscope_status pack_convg(const uint16_t* w, const ConvGGeom& g, uint8_t* out, cudaStream_t st) {
  const int64_t total = (int64_t)g.cout * g.steps * 16;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 4 * kNumSMs);
  pack_convg_kernel<<<grid, 256, 0, st>>>(w, g, reinterpret_cast<uint16_t*>(out));
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

NS_DEV uint16_t bf16_bits(float v) {
  __nv_bfloat16 h = __float2bfloat16_rn(v);
  return *reinterpret_cast<uint16_t*>(&h);
}

// Input normalisation (oracle normalize_input): x = clamp((g - mu_c)
// / 127.5, -1, 1) in fp32, rounded to bf16; channels 3..7 and separators zero.
__global__ void prep_sl_kernel(const uint8_t* __restrict__ small, int64_t pitch,
                               const int32_t* __restrict__ idx, const int64_t* __restrict__ n_dev,
                               int64_t n_max, int64_t chunk_base, int64_t chunk_len, float m0,
                               float m1, float m2, uint4* __restrict__ out) {
  const int64_t n = min(*n_dev, n_max);
  const int64_t cnt = min(n - chunk_base, chunk_len);
  if (cnt <= 0) return;
  constexpr int W = 50, Wq = 51, P = 51 * 51, G = 52;
  const int64_t total = G + cnt * P + Wq;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < total;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = make_uint4(0, 0, 0, 0);
    const int64_t rel = r - G;
    if (rel >= 0 && rel < cnt * P) {
      const int64_t f = rel / P;
      const int q = (int)(rel - f * P);
      const int Y = q / Wq, x = q - Y * Wq;
      if (Y >= 1 && x < W) {
        const int64_t gf = chunk_base + f;
        const int64_t fr = idx ? (int64_t)idx[gf] : gf;
        const uint8_t* px = small + fr * pitch + ((Y - 1) * W + x) * 3;
        const float a = fminf(fmaxf(((float)px[0] - m0) / 127.5f, -1.0f), 1.0f);
        const float b = fminf(fmaxf(((float)px[1] - m1) / 127.5f, -1.0f), 1.0f);
        const float c = fminf(fmaxf(((float)px[2] - m2) / 127.5f, -1.0f), 1.0f);
        v.x = (uint32_t)bf16_bits(a) | ((uint32_t)bf16_bits(b) << 16);
        v.y = bf16_bits(c);
      }
    }
    out[r] = v;
  }
}

noscope_status launch_prep_sl(const uint8_t* small, int64_t pitch, const int32_t* idx,
                              const int64_t* n_dev, int64_t n_max, int64_t chunk_base,
                              int64_t chunk_len, const float mean[3], uint8_t* out,
                              cudaStream_t st) {
  const int64_t rows = chunk_len * 51 * 51 + 52 + 51;
  const int grid = (int)std::min<int64_t>((rows + 255) / 256, 8 * kNumSMs);
  prep_sl_kernel<<<grid, 256, 0, st>>>(small, pitch, idx, n_dev, n_max, chunk_base, chunk_len,
                                       mean[0], mean[1], mean[2], reinterpret_cast<uint4*>(out));
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

__global__ void __launch_bounds__(gm::kThreads, 1)
convg_kernel(ConvGArgs A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const ConvGGeom& g = A.g;
  const int64_t n = min(*A.n_dev, A.n_max);
  const int64_t cnt = min(n - A.chunk_base, A.chunk_len);
  if (cnt <= 0) return;
  const int Wq = g.W + 1, P = (g.H + 1) * Wq, G = Wq + 1;
  const int64_t U = (cnt * P + g.S - 1) / g.S;
  if ((int64_t)blockIdx.x >= U) return;
  const int64_t my_units = (U - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncg = g.cin_eff / 8;
  const uint32_t plane = (uint32_t)g.rows_blk * 16;
  const uint32_t ablk = (uint32_t)ncg * plane;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.oBar);
  uint64_t* act_full = bars;           // [2]
  uint64_t* act_empty = bars + 2;      // [2]
  uint64_t* b_full = bars + 4;         // [8]
  uint64_t* b_empty = bars + 12;       // [8]
  uint64_t* acc_full = bars + 20;      // [2]
  uint64_t* acc_empty = bars + 22;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + gm::kNumBars);
  int* wcount = reinterpret_cast<int*>(tmem_slot + 1);
  float* bias = reinterpret_cast<float*>(smem + g.oBias);
  int2* wins = reinterpret_cast<int2*>(smem + g.oWin);

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&act_full[i], 1);
      mbar_init(&act_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], gm::kEpi / 32);
    }
    for (int i = 0; i < 8; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_rt(tmem_slot, g.tmem_cols);
  for (int c = tid; c < g.cout; c += blockDim.x) bias[c] = A.bias[c];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 10) {
    // ============================================== A producer
    if (lane == 0) {
      for (int64_t it = 0; it < my_units; ++it) {
        const int ab = (int)(it % g.nA);
        if (it >= g.nA) mbar_wait(&act_empty[ab], (uint32_t)(((it / g.nA) - 1) & 1));
        const int64_t u = blockIdx.x + it * gridDim.x;
        const int64_t r0 = (int64_t)G + u * g.S - Wq - 1;
        mbar_arrive_expect_tx(&act_full[ab], ablk);
        for (int c = 0; c < ncg; ++c)
          bulk_g2s(smem + (size_t)ab * ablk + (size_t)c * plane,
                   A.in + ((int64_t)c * g.R + r0) * 16, plane, &act_full[ab]);
      }
    }
  } else if (warp == 0) {
    // ============================================== B producer
    if (lane == 0) {
      const uint32_t bbytes = (uint32_t)g.N * 32;
      uint64_t seq = 0;
      for (int64_t it = 0; it < my_units; ++it)
        for (int p = 0; p < g.passes; ++p)
          for (int s = 0; s < g.steps; ++s, ++seq) {
            const int st = (int)(seq % g.bstages);
            if (seq >= (uint64_t)g.bstages)
              mbar_wait(&b_empty[st], (uint32_t)(((seq / g.bstages) - 1) & 1));
            mbar_arrive_expect_tx(&b_full[st], bbytes);
            bulk_g2s(smem + g.oB + (size_t)st * bbytes,
                     A.wpack + ((size_t)p * g.steps + s) * bbytes, bbytes, &b_full[st]);
          }
    }
  } else if (warp == 1) {
    // ============================================== MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(128, g.N);
      const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + g.oB);
      const uint32_t bbytes = (uint32_t)g.N * 32;
      uint64_t seq = 0, accseq = 0;
      for (int64_t it = 0; it < my_units; ++it) {
        const int ab = (int)(it % g.nA);
        mbar_wait(&act_full[ab], (uint32_t)((it / g.nA) & 1));
        tc_fence_after();
        const uint32_t aBase = sA + (uint32_t)ab * ablk + (uint32_t)(Wq + 1) * 16;
        for (int p = 0; p < g.passes; ++p, ++accseq) {
          const int b = (int)(accseq % g.nacc);
          if (accseq >= (uint64_t)g.nacc)
            mbar_wait(&acc_empty[b], (uint32_t)(((accseq / g.nacc) - 1) & 1));
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(b * g.MT * g.N);
          for (int s = 0; s < g.steps; ++s, ++seq) {
            const int st = (int)(seq % g.bstages);
            mbar_wait(&b_full[st], (uint32_t)((seq / g.bstages) & 1));
            tc_fence_after();
            int shift, lbo;
            uint32_t coff;
            if (g.cin_eff == 8) {   // two taps per K16 step
              const int t0 = 2 * s, t1 = 2 * s + 1;
              shift = (t0 / 3 - 1) * Wq + (t0 % 3 - 1);
              const int shift1 = t1 < 9 ? (t1 / 3 - 1) * Wq + (t1 % 3 - 1) : shift + 1;
              lbo = (shift1 - shift) * 16;
              coff = 0;
            } else {
              const int cpt = g.cin_eff / 16;
              const int tap = s / cpt;
              shift = (tap / 3 - 1) * Wq + (tap % 3 - 1);
              lbo = (int)plane;
              coff = (uint32_t)((s % cpt) * 2) * plane;
            }
            const uint64_t bd = sdesc(sB + (uint32_t)st * bbytes, (uint32_t)g.N * 16, 128);
            const uint32_t a0 = aBase + coff + (uint32_t)(shift * 16);
            for (int t = 0; t < g.MT; ++t)
              umma_bf16(d + (uint32_t)(t * g.N), sdesc(a0 + (uint32_t)t * 2048, (uint32_t)lbo, 128),
                        bd, idesc, s > 0 ? 1u : 0u);
            umma_commit(&b_empty[st]);
          }
          umma_commit(&acc_full[b]);
        }
        umma_commit(&act_empty[ab]);
      }
    }
  } else {
    // ============================================== epilogue (W2-W9)
    const int et = tid - 64;
    const int eg = (warp - 2) >> 2;      // tiles t = eg, eg + 2, ...
    const int lq = warp & 3;             // TMEM lane quarter of this warp
    const int Ho = g.H / 2, Wo = g.W / 2, Wqo = Wo + 1, Po = (Ho + 1) * Wqo, Go = Wqo + 1;
    const int ncg_out = g.cout / 8;
    if (blockIdx.x == 0 && !A.to_features) {  // zero the output's leading / trailing guards
      const int64_t tail0 = (int64_t)Go + cnt * Po;
      const int per = Go + Wqo;
      for (int e = et; e < ncg_out * per; e += gm::kEpi) {
        const int c = e / per, k = e % per;
        const int64_t row = k < Go ? k : tail0 + (k - Go);
        *reinterpret_cast<uint4*>(A.out + ((int64_t)c * A.out_rows + row) * 16) = make_uint4(0, 0, 0, 0);
      }
    }
    uint8_t* stage = smem + g.oStage;
    const uint32_t stage_bytes = (uint32_t)128 * g.MT * 32;
    uint64_t accseq = 0, slab = 0;
    for (int64_t it = 0; it < my_units; ++it) {
      const int64_t u = blockIdx.x + it * gridDim.x;
      const int64_t c0 = (int64_t)G + u * g.S;
      // ---- owned pool windows of this unit
      nbar_sync(1, gm::kEpi);
      if (et == 0) *wcount = 0;
      nbar_sync(1, gm::kEpi);
      for (int j = et; j < g.S; j += gm::kEpi) {
        const int64_t rel = c0 + j - G;
        const int64_t f = rel / P;
        if (f >= cnt) continue;
        const int q = (int)(rel - f * P);
        const int Y = q / Wq, x = q - Y * Wq, y = Y - 1;
        if (Y < 1 || (y & 1) || (x & 1) || (y >> 1) >= Ho || (x >> 1) >= Wo) continue;
        const int k = atomicAdd(wcount, 1);
        wins[k] = make_int2(j | ((y >> 1) << 16) | ((x >> 1) << 24), (int)f);
      }
      nbar_sync(1, gm::kEpi);
      const int nwin = *wcount;
      for (int p = 0; p < g.passes; ++p, ++accseq) {
        const int b = (int)(accseq % g.nacc);
        mbar_wait(&acc_full[b], (uint32_t)((accseq / g.nacc) & 1));
        tc_fence_after();
        const int nsl = g.N / 16;
        for (int sl = 0; sl < nsl; ++sl, ++slab) {
          uint8_t* sbuf = stage + (slab & 1) * stage_bytes;
          const int c = p * g.N + sl * 16;
          for (int t = eg; t < g.MT; t += 2) {
            uint32_t r[16];
            tmem_ld16(tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)((b * g.MT + t) * g.N + sl * 16), r);
            tmem_ld_wait();
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              pk[j] = relu_bf16x2(__uint_as_float(r[2 * j]) + bias[c + 2 * j],
                                  __uint_as_float(r[2 * j + 1]) + bias[c + 2 * j + 1]);
            uint4* dst = reinterpret_cast<uint4*>(sbuf + (size_t)(t * 128 + lq * 32 + lane) * 32);
            dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
          if (sl == nsl - 1) {  // accumulators fully read: release them to the MMA
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
          }
          nbar_sync(1, gm::kEpi);
          // ---- 2x2 max pool of the owned windows (non-negative bf16: integer max)
          for (int e = et; e < 2 * nwin; e += gm::kEpi) {
            const int2 w = wins[e >> 1];
            const int h = e & 1;
            const int sr = w.x & 0xFFFF, yp = (w.x >> 16) & 0xFF, xp = (w.x >> 24) & 0xFF;
            const int64_t f = w.y;
            const uint4* s0 = reinterpret_cast<const uint4*>(sbuf + (size_t)sr * 32) + h;
            const uint4 a0 = s0[0], a1 = s0[2], a2 = s0[2 * Wq], a3 = s0[2 * Wq + 2];
            uint4 o;
            o.x = __vmaxu2(__vmaxu2(a0.x, a1.x), __vmaxu2(a2.x, a3.x));
            o.y = __vmaxu2(__vmaxu2(a0.y, a1.y), __vmaxu2(a2.y, a3.y));
            o.z = __vmaxu2(__vmaxu2(a0.z, a1.z), __vmaxu2(a2.z, a3.z));
            o.w = __vmaxu2(__vmaxu2(a0.w, a1.w), __vmaxu2(a2.w, a3.w));
            const int cgo = c / 8 + h;
            if (A.to_features) {
              const int64_t kc = ((int64_t)(yp * Wo + xp) * g.cout) / 8 + cgo;
              *reinterpret_cast<uint4*>(A.out + (f / 128) * ((int64_t)A.K_feat * 256) + kc * 2048 +
                                        (f % 128) * 16) = o;
            } else {
              uint4* pl = reinterpret_cast<uint4*>(A.out + (int64_t)cgo * A.out_rows * 16);
              const int64_t orow = (int64_t)Go + f * Po + (int64_t)(yp + 1) * Wqo + xp;
              const uint4 z = make_uint4(0, 0, 0, 0);
              pl[orow] = o;
              if (xp == Wo - 1) pl[orow + 1] = z;           // separator column
              if (yp == 0) {                                  // separator row above
                pl[orow - Wqo] = z;
                if (xp == Wo - 1) pl[orow - Wqo + 1] = z;
              }
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc_rt(tmem, g.tmem_cols);
}

noscope_status launch_convg(const ConvGArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(convg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const ConvGGeom& g = a.g;
  const int64_t P = (int64_t)(g.H + 1) * (g.W + 1);
  const int64_t umax = (a.chunk_len * P + g.S - 1) / g.S;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(umax, kNumSMs));
  convg_kernel<<<grid, gm::kThreads, g.smem, st>>>(a);
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

}  // namespace ns
