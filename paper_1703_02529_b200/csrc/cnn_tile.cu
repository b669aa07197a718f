// cnn_tile.cu — the generic conv layer (cnn_gemm.cu) with 2-D M tiles for maps
// whose stacked row period H + 1 is even (conv2 of base_filters = 64: 25x25,
// Cout = 128).  An M tile is 8 consecutive columns x 16 consecutive image rows of
// the stacked space: 16 core-matrix groups one image row apart (SBO = Wq*16 B).
// A warp's 32 TMEM lanes then hold a 4-row x 8-column pixel block whose 2x2 pool
// windows are lane pairs (xor 1) and lane-octet pairs (xor 8): the epilogue pools
// with shuffles straight from registers — no shared-memory staging, so the
// tensor pipe's operand reads see no CUDA-core shared-memory traffic.  Because
// H + 1 is even, every frame's first image row has the same parity in the
// global row space, so 16-row blocks starting at odd global rows never split a
// pool window inside a frame.
//
// Unit = one 16-row block x XB column blocks (3 for 24 needed columns); the
// unit's A rows (18 image rows x Wq, two channel-group planes per stage) are
// streamed per channel-group pair, B per 3 taps (shared by the XB tiles), and
// the XB accumulators (N = 128 columns each) rotate through a 4-slot TMEM ring
// so the next unit's first tiles start while the epilogue drains the last ones.
#include "common.cuh"
#include "internal.h"

#ifndef NS_EXP
#define NS_EXP 0   // 256: per-role wait-time accounting (timing experiments only)
#endif
#if NS_EXP & 256
#include <algorithm>
#include <cstdio>
#include <vector>
#define NS_TT(k, stmt)                 \
  do {                                 \
    const long long _t0 = clock64();   \
    stmt;                              \
    twait[k] += clock64() - _t0;       \
  } while (0)
#else
#define NS_TT(k, stmt) stmt
#endif

namespace ns {

namespace gt {
constexpr int kThreads = 11 * 32;   // W0 B producer, W1 MMA, W2-W9 epilogue, W10 A producer
constexpr int kSlots = 4;           // TMEM accumulator slots of 128 columns
constexpr int kMaxA = 8, kMaxB = 24;
constexpr int kNumBars = 2 * kMaxA + 2 * kMaxB + 2 * kSlots;
}  // namespace gt

static size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool make_convt_geom(int cin, int cout, int H, int64_t chunk, ConvGGeom* out) {
  if (cin % 16 || cout != 128 || ((H + 1) & 1)) return false;
  ConvGGeom g{};
  g.tiled = 1;
  g.cin_real = g.cin_eff = cin;
  g.cout = cout;
  g.H = g.W = H;
  g.N = 128;
  g.passes = 1;
  g.steps = 9 * (cin / 16);
  g.MT = (2 * (H / 2) + 7) / 8;          // column blocks covering the pooled-map columns
  g.nacc = 1;
  const int Wq = H + 1;
  g.S = 16;                              // image rows per unit
  g.rows_blk = 18 * Wq + 2;
  g.R = sl_rows(H, H, chunk, 18 * Wq + 16);
  g.tmem_cols = 512;
  // B stage = 3 K16 steps (3 taps of one channel-group pair): one ring wait and
  // one completion commit per 3 x XB MMAs keeps the issuing thread ahead
  const size_t astage = (size_t)2 * g.rows_blk * 16, bstage = (size_t)3 * g.N * 32;
  auto layout = [&](int na, int nb) {
    size_t o = al((size_t)na * astage, 1024);
    g.oB = o;
    o = al(o + (size_t)nb * bstage, 128);
    g.oBias = o;
    o += (size_t)cout * 4;
    g.oBar = al(o, 8);
    o = g.oBar + gt::kNumBars * 8 + 16;
    return o + 1024;
  };
  g.nA = 4;
  g.kb = 3;
  g.bstages = 12;
  const size_t kMax = 227 * 1024;
  while (layout(g.nA, g.bstages) > kMax && g.bstages > 4) --g.bstages;
  g.smem = layout(g.nA, g.bstages);
  if (g.smem > kMax || g.MT > 3) return false;
  *out = g;
  return true;
}

__global__ void __launch_bounds__(gt::kThreads, 1)
convt_kernel(ConvGArgs A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const ConvGGeom& g = A.g;
  const int64_t n = min(*A.n_dev, A.n_max);
  const int64_t cnt = min(n - A.chunk_base, A.chunk_len);
  if (cnt <= 0) return;
  const int Wq = g.W + 1, Hp = g.H + 1, G = Wq + 1;
  const int64_t U = (cnt * Hp + 15) / 16;          // 16-row blocks over global image rows 1..cnt*Hp
  if ((int64_t)blockIdx.x >= U) return;
  const int64_t my_units = (U - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncgp = g.cin_eff / 16, XB = g.MT;
  const uint32_t plane = (uint32_t)g.rows_blk * 16, astage = 2 * plane;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.oBar);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + gt::kMaxA;
  uint64_t* b_full = a_empty + gt::kMaxA;
  uint64_t* b_empty = b_full + gt::kMaxB;
  uint64_t* t_full = b_empty + gt::kMaxB;     // [kSlots]
  uint64_t* t_empty = t_full + gt::kSlots;    // [kSlots] 4 epilogue-warp arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + gt::kNumBars);
  float* bias = reinterpret_cast<float*>(smem + g.oBias);

  if (tid == 0) {
    for (int i = 0; i < gt::kMaxA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < gt::kMaxB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < gt::kSlots; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  for (int c = tid; c < g.cout; c += blockDim.x) bias[c] = A.bias[c];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
#if NS_EXP & 256
  long long twait[8] = {};
  const long long tstart = clock64();
#endif

  if (warp == 10) {
    // ============================================== A producer
    if (lane == 0) {
      uint32_t st = 0, ph = 0, fill = 0;
      for (int64_t it = 0; it < my_units; ++it) {
        const int64_t u = blockIdx.x + it * gridDim.x;
        const int64_t r0 = (int64_t)G + 16 * u * Wq - 1;   // image row 16u, column -1
        for (int cp = 0; cp < ncgp; ++cp) {
          if (fill >= (uint32_t)g.nA) NS_TT(0, mbar_wait(&a_empty[st], ph ^ 1));
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
      const uint32_t bbytes = 3u * (uint32_t)g.N * 32;
      uint32_t st = 0, ph = 0, fill = 0;
      for (int64_t it = 0; it < my_units; ++it)
        for (int s = 0; s < g.steps; s += 3) {
          if (fill >= (uint32_t)g.bstages) NS_TT(1, mbar_wait(&b_empty[st], ph ^ 1));
          else ++fill;
          mbar_arrive_expect_tx(&b_full[st], bbytes);
          bulk_g2s(smem + g.oB + (size_t)st * bbytes, A.wpack + (size_t)s * (bbytes / 3), bbytes, &b_full[st]);
          if (++st == (uint32_t)g.bstages) { st = 0; ph ^= 1; }
        }
    }
  } else if (warp == 1) {
    // ============================================== MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(128, g.N);
      const uint32_t bstep = ((uint32_t)g.N * 32) >> 4;        // one K16 step of B
      const uint32_t bstage = 3 * bstep;
      const uint64_t bd0 = sdesc(smem_u32(smem + g.oB), (uint32_t)g.N * 16, 128);
      // tile (column block xb) at tap (ky, kx): block row offset ky*Wq + kx + 8*xb;
      // its 16 core-matrix groups are one image row (Wq*16 B) apart
      const uint64_t ad0 = sdesc(smem_u32(smem), plane, (uint32_t)Wq * 16);
      const uint32_t astep = astage >> 4;
      uint32_t ast = 0, aph = 0, bst = 0, bph = 0;
      uint32_t tseq = 0;   // global tile sequence -> TMEM slot tseq % 4
      for (int64_t it = 0; it < my_units; ++it, tseq += XB) {
        uint32_t col[3];
        for (int x = 0; x < XB; ++x) {
          const uint32_t t = tseq + x, sl = t % gt::kSlots;
          if (t >= (uint32_t)gt::kSlots) NS_TT(2, mbar_wait(&t_empty[sl], ((t / gt::kSlots) - 1) & 1u));
          col[x] = tmem + sl * 128;
        }
        tc_fence_after();
        for (int cp = 0; cp < ncgp; ++cp) {
          NS_TT(3, mbar_wait(&a_full[ast], aph));
          const uint64_t ac = ad0 + (uint64_t)(ast * astep);
#pragma unroll
          for (int ky = 0; ky < 3; ++ky) {          // B stage = taps (ky, 0..2)
            NS_TT(4, mbar_wait(&b_full[bst], bph));
            tc_fence_after();
            const uint64_t bs = bd0 + (uint64_t)(bst * bstage);
#pragma unroll
            for (int kx = 0; kx < 3; ++kx) {
              const uint64_t ad = ac + (uint64_t)(ky * Wq + kx);
              const uint64_t bd = bs + (uint64_t)(kx * bstep);
              const uint32_t acc = (cp | ky | kx) ? 1u : 0u;
              umma_bf16(col[0], ad, bd, idesc, acc);
              if (XB > 1) umma_bf16(col[1], ad + 8, bd, idesc, acc);   // +8 columns
              if (XB > 2) umma_bf16(col[2], ad + 16, bd, idesc, acc);
            }
            umma_commit(&b_empty[bst]);
            if (++bst == (uint32_t)g.bstages) { bst = 0; bph ^= 1; }
          }
          umma_commit(&a_empty[ast]);
          if (++ast == (uint32_t)g.nA) { ast = 0; aph ^= 1; }
        }
        for (int x = 0; x < XB; ++x) umma_commit(&t_full[(tseq + x) % gt::kSlots]);
      }
    }
  } else {
    // ============================================== epilogue (W2-W9)
    const int et = tid - 64;
    const int eg = (warp - 2) >> 2;               // tiles of the global sequence with t % 2 == eg
    const int lq = warp & 3;                      // TMEM lane quarter
    const int rl = lq * 4 + (lane >> 3), cl = lane & 7;   // row / column inside the tile
    const bool pool_lane = ((lane & 1) == 0) && (((lane >> 3) & 1) == 0);
    const int Ho = g.H / 2, Wo = g.W / 2, Wqo = Wo + 1, Po = (Ho + 1) * Wqo, Go = Wqo + 1;
    if (blockIdx.x == 0 && !A.to_features) {  // zero the output's leading / trailing guards
      const int64_t tail0 = (int64_t)Go + cnt * Po;
      const int per = Go + Wqo;
      for (int e = et; e < (g.cout / 8) * per; e += 256) {
        const int c = e / per, k = e % per;
        const int64_t row = k < Go ? k : tail0 + (k - Go);
        *reinterpret_cast<uint4*>(A.out + ((int64_t)c * A.out_rows + row) * 16) = make_uint4(0, 0, 0, 0);
      }
    }
    uint32_t tseq = 0;
    for (int64_t it = 0; it < my_units; ++it) {
      const int64_t u = blockIdx.x + it * gridDim.x;
      const int64_t Yg = 16 * u + 1 + rl;          // global image row of this lane
      const int64_t f = (Yg - 1) / Hp;
      const int y = (int)(Yg - 1 - f * Hp);
      for (int x = 0; x < XB; ++x, ++tseq) {
        if ((int)(tseq & 1) != eg) continue;
        const uint32_t sl = tseq % gt::kSlots;
        NS_TT(5, mbar_wait(&t_full[sl], (tseq / gt::kSlots) & 1u));
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(lq * 32) << 16) + sl * 128;
        uint32_t pk[64];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t r[32];
          tmem_ld16(ta + q * 32, *reinterpret_cast<uint32_t(*)[16]>(r));
          tmem_ld16(ta + q * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pk[q * 16 + j] = relu_bf16x2(__uint_as_float(r[2 * j]) + bias[q * 32 + 2 * j],
                                         __uint_as_float(r[2 * j + 1]) + bias[q * 32 + 2 * j + 1]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[sl]);   // accumulators free: next unit may start
#pragma unroll
        for (int j = 0; j < 64; ++j) {
          uint32_t v = pk[j];
          v = __vmaxu2(v, __shfl_xor_sync(0xffffffffu, v, 1));   // x pair
          v = __vmaxu2(v, __shfl_xor_sync(0xffffffffu, v, 8));   // y pair
          pk[j] = v;
        }
        const int xc = x * 8 + cl;
        const bool keep = pool_lane && f < cnt && y < 2 * Ho && xc < 2 * Wo;
        if (keep) {
          const int yp = y >> 1, xp = xc >> 1;
#pragma unroll
          for (int cg = 0; cg < 16; ++cg) {
            const uint4 o = make_uint4(pk[cg * 4], pk[cg * 4 + 1], pk[cg * 4 + 2], pk[cg * 4 + 3]);
            if (A.to_features) {
              const int64_t kc = ((int64_t)(yp * Wo + xp) * g.cout) / 8 + cg;
              *reinterpret_cast<uint4*>(A.out + (f / 128) * ((int64_t)A.K_feat * 256) + kc * 2048 +
                                        (f % 128) * 16) = o;
            } else {
              uint4* pl = reinterpret_cast<uint4*>(A.out + (int64_t)cg * A.out_rows * 16);
              const int64_t orow = (int64_t)Go + f * Po + (int64_t)(yp + 1) * Wqo + xp;
              const uint4 z = make_uint4(0, 0, 0, 0);
              pl[orow] = o;
              if (xp == Wo - 1) pl[orow + 1] = z;
              if (yp == 0) {
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
#if NS_EXP & 256
  twait[7] = clock64() - tstart;
  if (A.dbg && lane == 0)
    for (int k = 0; k < 8; ++k) A.dbg[((size_t)blockIdx.x * 11 + warp) * 8 + k] = twait[k];
#endif
  if (warp == 1) tmem_dealloc<512>(tmem);
}

noscope_status launch_convt(const ConvGArgs& a, cudaStream_t st) {
  static DeviceOnce attr;
  if (attr.first())
    NS_CUDA_TRY(cudaFuncSetAttribute(convt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  const ConvGGeom& g = a.g;
  const int64_t umax = (a.chunk_len * (g.H + 1) + 15) / 16;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(umax, kNumSMs));
#if NS_EXP & 256
  static long long* dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, (size_t)grid * 11 * 8 * 8);
  cudaMemset(dbg, 0, (size_t)grid * 11 * 8 * 8);
  ConvGArgs b = a;
  b.dbg = dbg;
  convt_kernel<<<grid, gt::kThreads, g.smem, st>>>(b);
  cudaDeviceSynchronize();
  {
    std::vector<long long> h((size_t)grid * 11 * 8);
    cudaMemcpy(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost);
    static const char* nm[8] = {"a_empty", "b_empty", "t_empty", "a_full", "b_full", "t_full", "-", "TOTAL"};
    for (int w = 0; w < 11; ++w) {
      long long tot = 0;
      for (int c = 0; c < grid; ++c) tot += h[((size_t)c * 11 + w) * 8 + 7];
      std::fprintf(stderr, "TT w%02d", w);
      for (int k = 0; k < 7; ++k) {
        long long sm = 0;
        for (int c = 0; c < grid; ++c) sm += h[((size_t)c * 11 + w) * 8 + k];
        if (sm) std::fprintf(stderr, " %s=%.1f%%", nm[k], 100.0 * sm / std::max(1ll, tot));
      }
      std::fprintf(stderr, "\n");
    }
  }
#else
  convt_kernel<<<grid, gt::kThreads, g.smem, st>>>(a);
#endif
  NS_LAUNCH_CHECK();
  count_launch();
  return NOSCOPE_OK;
}

}  // namespace ns
