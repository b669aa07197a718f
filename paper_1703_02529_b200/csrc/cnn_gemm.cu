// cnn_gemm.cu — one 3x3 conv + bias + ReLU + 2x2 max-pool layer of the
// specialized CNN (§4: "convolutional layers ... max
// pooling ... the number of filters doubles") as a batched implicit GEMM on
// tcgen05 tensor cores.  Used for every layer after the fused conv1(+conv2)
// kernel (cnn_fused.cu): conv2 of base_filters = 64 and conv3/conv4 of the
// 4-layer networks.
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
// K order: channel-group pair major, tap minor (s = cgp * 9 + tap), so both
// operands stream like an ordinary GEMM: A arrives one channel-group pair at a
// time (the unit's rows of 2 planes, re-read by the 9 taps), B one K16 step at a
// time; the ring depths are sized to cover L2 latency (weights are re-streamed
// per unit, so B is the bandwidth term).
//
// Roles (11 warps, persistent, one CTA per SM):
//   W10   A producer  — cp.async.bulk of the unit's rows of 2 channel-group planes
//                       per A stage
//   W0    B producer  — weight K-step slabs [2][N][8] through the B ring
//   W1    MMA issuer  — per pass over Cout: steps x MT tcgen05.mma (M=128, N,
//                       K=16), the MT tiles interleaved on independent
//                       accumulators; owns TMEM
//   W2-W9 epilogue    — TMEM -> +bias -> ReLU -> bf16 -> smem staging (32-channel
//                       slabs, double-buffered) -> 2x2 max of the owned windows
//                       -> next layer's stacked map (separators written as zeros)
//                       or the FC feature tiles
#include "common.cuh"
#include "internal.h"

namespace ns {

namespace gm {
constexpr int kThreads = 11 * 32;
constexpr int kEpi = 256;       // epilogue threads (W2-W9)
constexpr int kMaxWin = 256;    // owned pool windows per unit (<= S/4 + Wq)
constexpr int kMaxA = 8, kMaxB = 24;
constexpr int kNumBars = 2 * kMaxA + 2 * kMaxB + 2 + 2;
}  // namespace gm

static size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool make_convg_geom(int cin_real, int cout, int H, int64_t chunk, ConvGGeom* out) {
  ConvGGeom g{};
  g.cin_real = cin_real;
  g.cin_eff = cin_real;
  if (cin_real % 16) return false;
  g.cout = cout;
  g.H = H;
  g.W = H;
  // N = 256 per pass when Cout allows: B (re-streamed weights) is the traffic
  // term, and two 128-row tiles x 256 columns use all 512 TMEM columns.
  g.N = std::min(cout, 256);
  if (cout % g.N || g.N % 32) return false;
  g.passes = cout / g.N;
  g.steps = 9 * (g.cin_eff / 16);   // K16 steps: (channel-group pair, tap)
  g.MT = 2;
  g.nacc = 512 / (g.MT * g.N) >= 2 ? 2 : 1;
  const int Wq = g.W + 1;
  g.S = 128 * g.MT - Wq - 1;
  if (g.S <= 0) return false;
  g.rows_blk = 128 * g.MT + 2 * Wq + 2;   // [c0 - Wq - 1, c0 + 128 MT + Wq + 1)
  g.R = sl_rows(g.H, g.W, chunk, 128 * g.MT + Wq + 8);
  uint32_t tc = 32;
  while ((int)tc < g.nacc * g.MT * g.N) tc <<= 1;
  g.tmem_cols = tc;
  const size_t astage = (size_t)2 * g.rows_blk * 16;   // two channel-group planes
  // B stage = 3 K16 steps (taps (ky, 0..2) of one channel-group pair): one ring
  // wait + commit per 3 steps keeps the single issuing thread ahead of the pipe
  g.kb = 3;
  const size_t bstage = (size_t)g.kb * g.N * 32;
  auto layout = [&](int na, int nb) {
    size_t o = al((size_t)na * astage, 1024);
    g.oB = o;
    o = al(o + (size_t)nb * bstage, 128);
    g.oStage = o;
    o += (size_t)2 * 128 * g.MT * 64;   // staging: 2 x rows x 32 bf16
    g.oWin = o;
    o += (size_t)gm::kMaxWin * 8;
    g.oBias = o;
    o += (size_t)cout * 4;
    g.oBar = al(o, 8);
    o = g.oBar + gm::kNumBars * 8 + 16;
    return o + 1024;  // alignment slack
  };
  const size_t kMax = 227 * 1024;
  g.nA = 4;
  g.bstages = 12;
  while (layout(g.nA, g.bstages) > kMax && g.bstages > 4) --g.bstages;
  g.smem = layout(g.nA, g.bstages);
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
    const int tap = s % 9, ch = ((s / 9) * 2 + h) * 8 + e;
    out[t] = w[((int64_t)co * 9 + tap) * g.cin_real + ch];
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
  const int ncgp = g.cin_eff / 16;                 // channel-group pairs
  const uint32_t plane = (uint32_t)g.rows_blk * 16;
  const uint32_t astage = 2 * plane;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.oBar);
  uint64_t* a_full = bars;                   // [kMaxA]
  uint64_t* a_empty = a_full + gm::kMaxA;     // [kMaxA]
  uint64_t* b_full = a_empty + gm::kMaxA;     // [kMaxB]
  uint64_t* b_empty = b_full + gm::kMaxB;     // [kMaxB]
  uint64_t* acc_full = b_empty + gm::kMaxB;   // [2]
  uint64_t* acc_empty = acc_full + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + gm::kNumBars);
  int* wcount = reinterpret_cast<int*>(tmem_slot + 1);
  float* bias = reinterpret_cast<float*>(smem + g.oBias);
  int2* wins = reinterpret_cast<int2*>(smem + g.oWin);

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], gm::kEpi / 32);
    }
    for (int i = 0; i < gm::kMaxA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < gm::kMaxB; ++i) {
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
      uint32_t st = 0, ph = 0, fill = 0;
      for (int64_t it = 0; it < my_units; ++it) {
        const int64_t u = blockIdx.x + it * gridDim.x;
        const int64_t r0 = (int64_t)G + u * g.S - Wq - 1;
        for (int p = 0; p < g.passes; ++p)
          for (int cp = 0; cp < ncgp; ++cp) {
            if (fill >= (uint32_t)g.nA) mbar_wait(&a_empty[st], ph ^ 1);
            else ++fill;
            mbar_arrive_expect_tx(&a_full[st], astage);
            for (int h = 0; h < 2; ++h)
              bulk_g2s(smem + (size_t)st * astage + (size_t)h * plane,
                       A.in + ((int64_t)(2 * cp + h) * g.R + r0) * 16, plane, &a_full[st]);
            if (++st == (uint32_t)g.nA) { st = 0; ph ^= 1; }
          }
      }
    }
  } else if (warp == 0) {
    // ============================================== B producer
    if (lane == 0) {
      const uint32_t bbytes = (uint32_t)g.kb * (uint32_t)g.N * 32;
      uint32_t st = 0, ph = 0, fill = 0;
      for (int64_t it = 0; it < my_units; ++it)
        for (int p = 0; p < g.passes; ++p)
          for (int s = 0; s < g.steps; s += g.kb) {
            if (fill >= (uint32_t)g.bstages) mbar_wait(&b_empty[st], ph ^ 1);
            else ++fill;
            mbar_arrive_expect_tx(&b_full[st], bbytes);
            bulk_g2s(smem + g.oB + (size_t)st * bbytes,
                     A.wpack + ((size_t)p * g.steps + s) * (bbytes / g.kb), bbytes, &b_full[st]);
            if (++st == (uint32_t)g.bstages) { st = 0; ph ^= 1; }
          }
    }
  } else if (warp == 1) {
    // ============================================== MMA issuer
    // The single issuing thread must stay far ahead of the tensor pipe: per
    // step one ring wait, two descriptor adds and MT tcgen05.mma; the 9 tap
    // offsets are loop constants, rings advance incrementally.
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(128, g.N);
      const uint32_t sB = smem_u32(smem + g.oB);
      const uint32_t bstep = ((uint32_t)g.N * 32) >> 4;   // one K16 step of B
      const uint32_t bstage = (uint32_t)g.kb * bstep;
      const uint64_t bd0 = sdesc(sB, (uint32_t)g.N * 16, 128);
      const uint64_t ad0 = sdesc(smem_u32(smem) + (uint32_t)(Wq + 1) * 16, plane, 128);
      const uint32_t astep = astage >> 4;
      uint64_t dtap[9];
#pragma unroll
      for (int t = 0; t < 9; ++t) dtap[t] = (uint64_t)(int64_t)((t / 3 - 1) * Wq + (t % 3 - 1));
      const uint32_t acol = (uint32_t)g.N;
      uint32_t ast = 0, aph = 0, bst = 0, bph = 0, accseq = 0;
      const int lgacc = g.nacc == 2 ? 1 : 0;
      for (int64_t it = 0; it < my_units; ++it) {
        for (int p = 0; p < g.passes; ++p, ++accseq) {
          const uint32_t b = accseq & (uint32_t)(g.nacc - 1);
          if (accseq >= (uint32_t)g.nacc)
            mbar_wait(&acc_empty[b], ((accseq >> lgacc) - 1) & 1u);
          tc_fence_after();
          const uint32_t d = tmem + b * (uint32_t)g.MT * acol;
          for (int cp = 0; cp < ncgp; ++cp) {
            mbar_wait(&a_full[ast], aph);
            const uint64_t ac = ad0 + (uint64_t)(ast * astep);
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {        // B stage = taps (ky, 0..2)
              mbar_wait(&b_full[bst], bph);
              tc_fence_after();
              const uint64_t bs = bd0 + (uint64_t)(bst * bstage);
#pragma unroll
              for (int kx = 0; kx < 3; ++kx) {
                const int t = ky * 3 + kx;
                const uint64_t ad = ac + dtap[t];
                const uint64_t bd = bs + (uint64_t)(kx * bstep);
                const uint32_t acc = (cp | t) ? 1u : 0u;
                umma_bf16(d, ad, bd, idesc, acc);
                umma_bf16(d + acol, ad + 128, bd, idesc, acc);   // +2048 B = next 128 rows
              }
              umma_commit(&b_empty[bst]);
              if (++bst == (uint32_t)g.bstages) { bst = 0; bph ^= 1; }
            }
            umma_commit(&a_empty[ast]);
            if (++ast == (uint32_t)g.nA) { ast = 0; aph ^= 1; }
          }
          umma_commit(&acc_full[b]);
        }
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
    const uint32_t stage_bytes = (uint32_t)128 * g.MT * 64;
    uint32_t accseq = 0, slab = 0;
    for (int64_t it = 0; it < my_units; ++it) {
      const int64_t u = blockIdx.x + it * gridDim.x;
      const int64_t c0 = (int64_t)G + u * g.S;
      // ---- owned pool windows of this unit
      nbar_sync(1, gm::kEpi);
      if (et == 0) *wcount = 0;
      nbar_sync(1, gm::kEpi);
      for (int j = et; j < g.S; j += gm::kEpi) {
        const int rel = (int)(c0 + j - G);   // < chunk * P < 2^31
        const int f = rel / P;
        if (f >= cnt) continue;
        const int q = rel - f * P;
        const int Y = q / Wq, x = q - Y * Wq, y = Y - 1;
        if (Y < 1 || (y & 1) || (x & 1) || (y >> 1) >= Ho || (x >> 1) >= Wo) continue;
        const int k = atomicAdd(wcount, 1);
        wins[k] = make_int2(j | ((y >> 1) << 16) | ((x >> 1) << 24), f);
      }
      nbar_sync(1, gm::kEpi);
      const int nwin = *wcount;
      for (int p = 0; p < g.passes; ++p, ++accseq) {
        const uint32_t b = accseq & (uint32_t)(g.nacc - 1);
        mbar_wait(&acc_full[b], (accseq >> (g.nacc == 2 ? 1 : 0)) & 1u);
        tc_fence_after();
        const int nsl = g.N / 32;
        for (int sl = 0; sl < nsl; ++sl, ++slab) {
          uint8_t* sbuf = stage + (slab & 1) * stage_bytes;
          const int c = p * g.N + sl * 32;
          for (int t = eg; t < g.MT; t += 2) {
            uint32_t r[32];
            const uint32_t ta = tmem + ((uint32_t)(lq * 32) << 16) + (b * g.MT + t) * (uint32_t)g.N + sl * 32;
            tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(r));
            tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              pk[j] = relu_bf16x2(__uint_as_float(r[2 * j]) + bias[c + 2 * j],
                                  __uint_as_float(r[2 * j + 1]) + bias[c + 2 * j + 1]);
            // 16-B chunk q of row r lives at chunk q ^ ((r >> 1) & 3): the 8 rows of a
            // 128-B wavefront then hit 8 distinct bank groups (no 4-way conflicts)
            const int row = t * 128 + lq * 32 + lane;
            uint4* dst = reinterpret_cast<uint4*>(sbuf + (size_t)row * 64);
            const int sw = (row >> 1) & 3;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              dst[q ^ sw] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
          if (sl == nsl - 1) {  // accumulators fully read: release them to the MMA
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
          }
          nbar_sync(1, gm::kEpi);
          // ---- 2x2 max pool of the owned windows (non-negative bf16: integer max)
          for (int e = et; e < 4 * nwin; e += gm::kEpi) {
            const int2 w = wins[e >> 2];
            const int h = e & 3;
            const int sr = w.x & 0xFFFF, yp = (w.x >> 16) & 0xFF, xp = (w.x >> 24) & 0xFF;
            const int64_t f = w.y;
            const uint4* sb4 = reinterpret_cast<const uint4*>(sbuf);
            auto at = [&](int r) { return sb4[r * 4 + (h ^ ((r >> 1) & 3))]; };   // swizzled chunk
            const uint4 a0 = at(sr), a1 = at(sr + 1), a2 = at(sr + Wq), a3 = at(sr + Wq + 1);
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
  static DeviceOnce attr;
  if (attr.first())
    NS_CUDA_TRY(cudaFuncSetAttribute(convg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
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
