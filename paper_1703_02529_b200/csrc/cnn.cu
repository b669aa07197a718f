// cnn.cu — the specialized CNN (§4; north star: "3x3
// conv+ReLU+maxpool layers, a dense layer and a sigmoid") on tcgen05 tensor
// cores: bf16 operands from shared memory, fp32 accumulators in TMEM.
//
// Layer 1 (Cin = 3): explicit im2col tile per 128 output pixels, K = 27 padded
//   to 32 (two K=16 MMAs).  Rows are ordered pool-window-major (4 consecutive
//   rows = one 2x2 pool window), so bias+ReLU+maxpool happen in registers with
//   two warp shuffles straight out of TMEM.  The fp32->bf16 normalisation
//    is fused into the input load.
// Layers 2..L: "shifted-window" implicit GEMM.  The haloed input map of a
//   frame lives in shared memory as Cin/8 planes of [row q = yy*Wp + xx][8 ch]
//   (16 B per row) = exactly the canonical K-major no-swizzle UMMA layout, so
//   the A operand of tap (ty, tx) for an M tile starting at row q0 is just a
//   descriptor whose start address is shifted by ((ty-1)*Wp + tx-1) rows: no
//   im2col is materialised and all 9 taps read the same smem.  B (weights) is
//   streamed through a 4-stage cp.async.bulk ring.  Epilogue: TMEM -> bias ->
//   ReLU -> bf16 -> smem staging -> 2x2 max (integer max of non-negative bf16
//   bit patterns) -> next layer's haloed map (or the FC feature matrix).
// FC: features (h, w, c) in the canonical A layout [tile][K/8][128][8] ->
//   tcgen05 GEMM with N = dense, epilogue bias+ReLU+bf16, FC2 dot + bias.
#include "common.cuh"
#include "internal.h"

namespace ns {

constexpr int kCnnThreads = 128;
constexpr int kBStages = 4;
constexpr int64_t kCnnChunk = 8192;   // frames per internal chunk (workspace bound)
constexpr int kIn = 50, kInP = 52, kP1 = 25, kHp2 = 27;
constexpr int kInBytes = 7504;  // 50*50*3 rounded up to 16
constexpr int kInBytes_ = kInBytes;

NS_DEV uint16_t f2bf(float v) {
  __nv_bfloat16 h = __float2bfloat16_rn(v);
  return *reinterpret_cast<uint16_t*>(&h);
}
NS_DEV float bf2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

static uint32_t tmem_cols_host(int c) {
  uint32_t r = 32;
  while ((int)r < c) r <<= 1;
  return r;
}
template <int C>
constexpr size_t conv1_smem_bytes() {
  return 16384 + 2 * kInBytes_ + 52 * 52 * 3 * 2 + 4 * C * 16 + C * 4 + 4 * 8 + 16;
}

// Runtime TMEM alloc (power of two >= 32 columns), whole warp.
NS_DEV void tmem_alloc_rt(uint32_t* dst, uint32_t cols) {
  switch (cols) {
    case 32: tmem_alloc<32>(dst); break;
    case 64: tmem_alloc<64>(dst); break;
    case 128: tmem_alloc<128>(dst); break;
    case 256: tmem_alloc<256>(dst); break;
    default: tmem_alloc<512>(dst); break;
  }
}
NS_DEV void tmem_dealloc_rt(uint32_t taddr, uint32_t cols) {
  switch (cols) {
    case 32: tmem_dealloc<32>(taddr); break;
    case 64: tmem_dealloc<64>(taddr); break;
    case 128: tmem_dealloc<128>(taddr); break;
    case 256: tmem_dealloc<256>(taddr); break;
    default: tmem_dealloc<512>(taddr); break;
  }
}

// ------------------------------------------------------------ weight packing
// out[((p*nkc + kc)*pn + n)*8 + e] = w[(p*pn + n)*Kreal + kc*8 + e] (0 beyond Kreal)
__global__ void pack_kernel(const uint16_t* __restrict__ w, int rows, int Kreal, int Kpad, int pn,
                            uint16_t* __restrict__ out) {
  const int nkc = Kpad / 8;
  const int64_t total = (int64_t)rows * Kpad;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t & 7);
    const int64_t r = t >> 3;
    const int n_all = (int)(r % rows);
    const int kc = (int)(r / rows);
    const int p = n_all / pn, n = n_all % pn;
    const int k = kc * 8 + e;
    out[(((int64_t)p * nkc + kc) * pn + n) * 8 + e] = k < Kreal ? w[(int64_t)n_all * Kreal + k] : 0;
  }
}

// =================================================================== layer 1
struct Conv1Args {
  const uint8_t* small;
  int64_t small_pitch;
  const int32_t* idx;
  const int64_t* n_dev;
  int64_t n_max, chunk_base, chunk_len;
  const uint16_t* wpack;  // [4 kc][C][8]
  const float* bias;
  float mean[3];
  uint8_t* act_out;       // [chunk][C/8][27*27][16 B]
  int64_t out_frame_bytes;
};


template <int C>
__global__ void __launch_bounds__(kCnnThreads)
conv1_kernel(Conv1Args A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // dynamic smem carve-up (see conv1_smem_bytes)
  uint8_t (*Abuf)[128 * 64] = reinterpret_cast<uint8_t (*)[128 * 64]>(smem);          // 16 KB
  uint8_t (*in_u8)[kInBytes] = reinterpret_cast<uint8_t (*)[kInBytes]>(smem + 16384); // 2 x 7504
  uint16_t* X = reinterpret_cast<uint16_t*>(smem + 16384 + 2 * kInBytes);             // 52*52*3
  uint8_t* Bs = smem + 16384 + 2 * kInBytes + kInP * kInP * 3 * 2;                    // 4*C*16
  float* bias_s = reinterpret_cast<float*>(Bs + 4 * C * 16);
  uint64_t* bar_in = reinterpret_cast<uint64_t*>(bias_s + C);
  uint64_t* bar_mma = bar_in + 2;
  uint32_t* tmem_base_p = reinterpret_cast<uint32_t*>(bar_mma + 2);

  const int64_t n = min(*A.n_dev, A.n_max);
  const int64_t cnt = min(n - A.chunk_base, A.chunk_len);
  if (cnt <= 0 || blockIdx.x >= cnt) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t kCols = 2 * C;

  if (tid == 0) {
    mbar_init(&bar_in[0], 1);
    mbar_init(&bar_in[1], 1);
    mbar_init(&bar_mma[0], 1);
    mbar_init(&bar_mma[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<kCols>(tmem_base_p);
  for (int t = tid; t < 4 * C * 8; t += blockDim.x)
    reinterpret_cast<uint16_t*>(Bs)[t] = A.wpack[t];
  for (int t = tid; t < C; t += blockDim.x) bias_s[t] = A.bias[t];
  for (int t = tid; t < kInP * kInP * 3; t += blockDim.x) X[t] = 0;  // zero halo
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_p;

  auto frame_ptr = [&](int64_t i) {
    const int64_t g = A.chunk_base + i;
    const int64_t f = A.idx ? (int64_t)A.idx[g] : g;
    return A.small + f * A.small_pitch;
  };
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_in[0], kInBytes);
    bulk_g2s(in_u8[0], frame_ptr(blockIdx.x), kInBytes, &bar_in[0]);
  }
  constexpr uint32_t idesc = idesc_bf16_f32(128, C);
  uint32_t ts = 0;  // global tile sequence (A buffer / TMEM half / mbarrier parity)
  int it = 0;
  for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x, ++it) {
    const int b = it & 1;
    mbar_wait(&bar_in[b], (uint32_t)((it >> 1) & 1));
    if (tid == 0 && i + gridDim.x < cnt) {
      mbar_arrive_expect_tx(&bar_in[b ^ 1], kInBytes);
      bulk_g2s(in_u8[b ^ 1], frame_ptr(i + gridDim.x), kInBytes, &bar_in[b ^ 1]);
    }
    // normalise: x = bf16(clamp((G - mu_c) / 127.5, -1, 1))
    for (int e = tid; e < kIn * kIn * 3; e += blockDim.x) {
      const int p = e / 3, c = e - 3 * p;
      const int y = p / kIn, x = p - kIn * y;
      float v = ((float)in_u8[b][e] - A.mean[c]) / 127.5f;
      v = fminf(fmaxf(v, -1.0f), 1.0f);
      X[((y + 1) * kInP + (x + 1)) * 3 + c] = f2bf(v);
    }
    // zero this frame's output halo ring
    uint8_t* outf = A.act_out + i * A.out_frame_bytes;
    for (int e = tid; e < (C / 8) * 4 * (kHp2 - 1); e += blockDim.x) {
      const int cg = e / (4 * (kHp2 - 1)), h = e % (4 * (kHp2 - 1));
      const int side = h / (kHp2 - 1), s = h % (kHp2 - 1);
      int yy, xx;
      if (side == 0) { yy = 0; xx = s; }
      else if (side == 1) { yy = s; xx = kHp2 - 1; }
      else if (side == 2) { yy = kHp2 - 1; xx = s + 1; }
      else { yy = s + 1; xx = 0; }
      *reinterpret_cast<uint4*>(outf + (size_t)cg * kHp2 * kHp2 * 16 + (yy * kHp2 + xx) * 16) =
          make_uint4(0, 0, 0, 0);
    }
    __syncthreads();

    constexpr int kTiles = (kP1 * kP1 * 4 + 127) / 128;  // 20
    for (int t = 0; t < kTiles; ++t, ++ts) {
      const int ab = ts & 1;
      // ---- build im2col row m = tid (pool-window-major ordering)
      {
        const int w = t * 32 + (tid >> 2), pq = tid & 3;
        uint16_t v[32];
        if (w < kP1 * kP1) {
          const int yp = w / kP1, xp = w - kP1 * yp;
          const int y = 2 * yp + (pq >> 1), x = 2 * xp + (pq & 1);
#pragma unroll
          for (int ky = 0; ky < 3; ++ky)
#pragma unroll
            for (int kx = 0; kx < 3; ++kx)
#pragma unroll
              for (int c = 0; c < 3; ++c)
                v[(ky * 3 + kx) * 3 + c] = X[((y + ky) * kInP + (x + kx)) * 3 + c];
        } else {
#pragma unroll
          for (int k = 0; k < 27; ++k) v[k] = 0;
        }
#pragma unroll
        for (int k = 27; k < 32; ++k) v[k] = 0;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          uint4 q;
          q.x = v[kc * 8 + 0] | ((uint32_t)v[kc * 8 + 1] << 16);
          q.y = v[kc * 8 + 2] | ((uint32_t)v[kc * 8 + 3] << 16);
          q.z = v[kc * 8 + 4] | ((uint32_t)v[kc * 8 + 5] << 16);
          q.w = v[kc * 8 + 6] | ((uint32_t)v[kc * 8 + 7] << 16);
          *reinterpret_cast<uint4*>(&Abuf[ab][kc * 2048 + tid * 16]) = q;
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t a0 = smem_u32(&Abuf[ab][0]), b0 = smem_u32(Bs);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          umma_bf16(tmem + ab * C, sdesc(a0 + kk * 2 * 2048, 2048, 128),
                    sdesc(b0 + kk * 2 * C * 16, C * 16, 128), idesc, kk);
        umma_commit(&bar_mma[ab]);
      }
      // ---- epilogue of this tile
      mbar_wait(&bar_mma[ab], (ts >> 1) & 1);
      tc_fence_after();
      const int w = t * 32 + (tid >> 2);
      const bool valid = w < kP1 * kP1 && (lane & 3) == 0;
      const int yp = w / kP1, xp = w - kP1 * (w / kP1);
#pragma unroll
      for (int cb = 0; cb < C / 16; ++cb) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + ab * C + cb * 16, r);
        tmem_ld_wait();
        uint32_t packed[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          float v0 = fmaxf(__uint_as_float(r[j]) + bias_s[cb * 16 + j], 0.0f);
          float v1 = fmaxf(__uint_as_float(r[j + 1]) + bias_s[cb * 16 + j + 1], 0.0f);
          v0 = fmaxf(v0, __shfl_xor_sync(0xffffffffu, v0, 1));
          v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, 1));
          v0 = fmaxf(v0, __shfl_xor_sync(0xffffffffu, v0, 2));
          v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, 2));
          packed[j >> 1] = (uint32_t)f2bf(v0) | ((uint32_t)f2bf(v1) << 16);
        }
        if (valid) {
          const size_t pix = (size_t)((yp + 1) * kHp2 + (xp + 1)) * 16;
          const int cg = cb * 2;
          *reinterpret_cast<uint4*>(outf + (size_t)cg * kHp2 * kHp2 * 16 + pix) =
              make_uint4(packed[0], packed[1], packed[2], packed[3]);
          *reinterpret_cast<uint4*>(outf + (size_t)(cg + 1) * kHp2 * kHp2 * 16 + pix) =
              make_uint4(packed[4], packed[5], packed[6], packed[7]);
        }
      }
      tc_fence_before();
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<kCols>(tmem);
}

// =================================================================== layers 2..L
struct ConvNArgs {
  const uint8_t* act_in;
  int64_t in_frame_bytes;
  int cin, hp, wp;            // input haloed map
  uint8_t* act_out;
  int64_t out_frame_bytes;
  int hp_out, wp_out;
  uint8_t* feat;              // last layer: FC feature matrix (canonical A layout)
  int K_feat;
  int last;
  const uint8_t* wpack;       // [pass][kc][pass_n][8]
  const float* bias;
  int cout, hpool;
  int n_tiles, n_pass, pass_n, mma_n, chunk_ch, chunks_per_pass, chunk_bytes;
  int plane_rows;             // rows per smem plane (q = -1 .. )
  uint32_t tmem_cols;
  const int64_t* n_dev;
  int64_t n_max, chunk_base, chunk_len;
};

constexpr int kEpCols = 16;  // epilogue column group (2 channel groups)

__global__ void __launch_bounds__(kCnnThreads, 1)
convN_kernel(ConvNArgs A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int64_t n = min(*A.n_dev, A.n_max);
  const int64_t cnt = min(n - A.chunk_base, A.chunk_len);
  if (cnt <= 0 || blockIdx.x >= cnt) return;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncg = A.cin / 8;
  const uint32_t plane_bytes = (uint32_t)A.plane_rows * 16;
  uint8_t* planes = smem;                                           // ncg * plane_bytes
  uint8_t* bstage = planes + (((size_t)ncg * plane_bytes + 1023) & ~(size_t)1023);
  uint8_t* staging = bstage + (size_t)kBStages * A.chunk_bytes;     // n_tiles*128 rows * 32 B
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + (size_t)A.n_tiles * 128 * kEpCols * 2);
  uint64_t* full = bars;                 // [kBStages]
  uint64_t* empty = bars + kBStages;     // [kBStages]
  uint64_t* bar_a = bars + 2 * kBStages; // A planes loaded
  uint64_t* bar_acc = bar_a + 1;         // accumulators ready
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(bar_acc + 1);

  if (tid == 0) {
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(bar_a, 1);
    mbar_init(bar_acc, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_rt(tmem_s, A.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_s;

  const int chunks_total = A.n_pass * A.chunks_per_pass;  // per frame
  const uint32_t idesc = idesc_bf16_f32(128, A.mma_n);
  const uint32_t planes_s = smem_u32(planes), bstage_s = smem_u32(bstage);
  const int in_rows = A.hp * A.wp;

  // producer state (thread 0): global chunk sequence across frames
  uint64_t load_seq = 0, mma_seq = 0;
  const int64_t my_frames = (cnt - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint64_t total_chunks = (uint64_t)my_frames * chunks_total;
  auto issue_b = [&](uint64_t s) {
    const int stage = (int)(s % kBStages);
    const int c = (int)(s % chunks_total);
    if (s >= kBStages) mbar_wait(&empty[stage], (uint32_t)(((s / kBStages) - 1) & 1));
    mbar_arrive_expect_tx(&full[stage], A.chunk_bytes);
    bulk_g2s(bstage + (size_t)stage * A.chunk_bytes, A.wpack + (size_t)c * A.chunk_bytes,
             A.chunk_bytes, &full[stage]);
  };
  if (tid == 0)
    for (; load_seq < (uint64_t)kBStages - 1 && load_seq < total_chunks; ++load_seq) issue_b(load_seq);

  int it = 0;
  uint32_t acc_phase = 0;
  for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x, ++it) {
    // ---- load the haloed input map: one bulk copy per channel-group plane
    if (tid == 0) {
      const uint8_t* src = A.act_in + i * A.in_frame_bytes;
      mbar_arrive_expect_tx(bar_a, (uint32_t)(ncg * in_rows * 16));
      for (int cg = 0; cg < ncg; ++cg)
        bulk_g2s(planes + (size_t)cg * plane_bytes + 16, src + (size_t)cg * in_rows * 16,
                 in_rows * 16, bar_a);
    }
    // zero the output halo ring of this frame (non-last layers)
    if (!A.last) {
      uint8_t* outf = A.act_out + i * A.out_frame_bytes;
      const int ring = 4 * (A.hp_out - 1);
      const int ncg_out = A.cout / 8;
      for (int e = tid; e < ncg_out * ring; e += blockDim.x) {
        const int cg = e / ring, h = e % ring;
        const int side = h / (A.hp_out - 1), s = h % (A.hp_out - 1);
        int yy, xx;
        if (side == 0) { yy = 0; xx = s; }
        else if (side == 1) { yy = s; xx = A.wp_out - 1; }
        else if (side == 2) { yy = A.hp_out - 1; xx = s + 1; }
        else { yy = s + 1; xx = 0; }
        *reinterpret_cast<uint4*>(outf + (size_t)cg * A.hp_out * A.wp_out * 16 +
                                  (size_t)(yy * A.wp_out + xx) * 16) = make_uint4(0, 0, 0, 0);
      }
    }
    mbar_wait(bar_a, (uint32_t)(it & 1));

    for (int p = 0; p < A.n_pass; ++p) {
      // ---- MMA issue (thread 0): all chunks of this pass, all M tiles
      if (tid == 0) {
        tc_fence_after();
        for (int c = 0; c < A.chunks_per_pass; ++c, ++mma_seq) {
          const int stage = (int)(mma_seq % kBStages);
          mbar_wait(&full[stage], (uint32_t)((mma_seq / kBStages) & 1));
          tc_fence_after();
          const int k0 = c * A.chunk_ch;              // first channel of K in (tap, ch) order
          const int tap = k0 / A.cin, cg0 = (k0 % A.cin) / 8;
          const int shift = (tap / 3 - 1) * A.wp + (tap % 3 - 1);
          const uint32_t bs = bstage_s + (uint32_t)stage * A.chunk_bytes;
          for (int kk = 0; kk < A.chunk_ch / 16; ++kk) {
            const int cg = cg0 + 2 * kk;
            for (int t = 0; t < A.n_tiles; ++t) {
              const int q0 = A.wp + t * 128;
              const uint32_t a_addr =
                  planes_s + (uint32_t)cg * plane_bytes + (uint32_t)(q0 + shift + 1) * 16;
              const uint64_t ad = sdesc(a_addr, plane_bytes, 128);
              for (int nh = 0; nh < A.pass_n / A.mma_n; ++nh) {
                const uint64_t bd =
                    sdesc(bs + (uint32_t)(2 * kk) * A.pass_n * 16 + nh * A.mma_n * 16,
                          A.pass_n * 16, 128);
                umma_bf16(tmem + t * A.pass_n + nh * A.mma_n, ad, bd, idesc,
                          (c > 0 || kk > 0) ? 1u : 0u);
              }
            }
          }
          umma_commit(&empty[stage]);
          if (load_seq < total_chunks) issue_b(load_seq++);
        }
        umma_commit(bar_acc);
      }
      __syncwarp();
      // ---- epilogue
      mbar_wait(bar_acc, acc_phase);
      acc_phase ^= 1;
      tc_fence_after();
      const int ncg_out = A.cout / 8;
      for (int cgp = 0; cgp < A.pass_n / kEpCols; ++cgp) {
        for (int t = 0; t < A.n_tiles; ++t) {
          uint32_t r[16];
          tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + t * A.pass_n + cgp * kEpCols, r);
          tmem_ld_wait();
          const int ch0 = p * A.pass_n + cgp * kEpCols;
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float v0 = relu(__uint_as_float(r[j]) + A.bias[ch0 + j]);
            const float v1 = relu(__uint_as_float(r[j + 1]) + A.bias[ch0 + j + 1]);
            pk[j >> 1] = (uint32_t)f2bf(v0) | ((uint32_t)f2bf(v1) << 16);
          }
          uint4* dst = reinterpret_cast<uint4*>(staging + (size_t)(t * 128 + tid) * 32);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        __syncthreads();
        // 2x2 max pool of the staged rows -> outputs
        const int npix = A.hpool * A.hpool;
        for (int e = tid; e < npix * 2; e += blockDim.x) {
          const int half = e & 1, pix = e >> 1;
          const int yp = pix / A.hpool, xp = pix % A.hpool;
          const int r0 = (2 * yp + 1) * A.wp + (2 * xp + 1) - A.wp;  // staging row of (2y'+1, 2x'+1)
          const uint4* s0 = reinterpret_cast<const uint4*>(staging + (size_t)r0 * 32) + half;
          const uint4* s1 = reinterpret_cast<const uint4*>(staging + (size_t)(r0 + 1) * 32) + half;
          const uint4* s2 = reinterpret_cast<const uint4*>(staging + (size_t)(r0 + A.wp) * 32) + half;
          const uint4* s3 =
              reinterpret_cast<const uint4*>(staging + (size_t)(r0 + A.wp + 1) * 32) + half;
          uint4 a = *s0, b = *s1, c = *s2, d = *s3, o;
          o.x = __vmaxu2(__vmaxu2(a.x, b.x), __vmaxu2(c.x, d.x));
          o.y = __vmaxu2(__vmaxu2(a.y, b.y), __vmaxu2(c.y, d.y));
          o.z = __vmaxu2(__vmaxu2(a.z, b.z), __vmaxu2(c.z, d.z));
          o.w = __vmaxu2(__vmaxu2(a.w, b.w), __vmaxu2(c.w, d.w));
          const int cgo = (p * A.pass_n + cgp * kEpCols) / 8 + half;
          if (!A.last) {
            uint8_t* outf = A.act_out + i * A.out_frame_bytes;
            *reinterpret_cast<uint4*>(outf + (size_t)cgo * A.hp_out * A.wp_out * 16 +
                                      (size_t)((yp + 1) * A.wp_out + (xp + 1)) * 16) = o;
          } else {
            const int64_t kc = ((int64_t)(yp * A.hpool + xp) * A.cout) / 8 + cgo;
            *reinterpret_cast<uint4*>(A.feat + (i / 128) * ((int64_t)A.K_feat * 256) +
                                      kc * 2048 + (i % 128) * 16) = o;
          }
        }
        (void)ncg_out;
        __syncthreads();
      }
      tc_fence_before();
      __syncthreads();
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc_rt(tmem, A.tmem_cols);
}

// =================================================================== FC
struct FcArgs {
  const uint8_t* feat;   // [tiles][K/8][128][8] bf16
  int K, D;
  const uint8_t* wpack;  // [K/8][D][8] bf16
  const float* b1;
  const uint16_t* w2;
  const float* b2;
  float* logits;
  const int64_t* n_dev;
  int64_t n_max, chunk_base, chunk_len;
  uint32_t tmem_cols;
};
constexpr int kFcKChunk = 64;

__global__ void __launch_bounds__(kCnnThreads)
fc_kernel(FcArgs A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int64_t n = min(*A.n_dev, A.n_max);
  const int64_t cnt = min(n - A.chunk_base, A.chunk_len);
  const int64_t tile = blockIdx.x;
  if (cnt <= 0 || tile * 128 >= cnt) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t a_bytes = 128 * kFcKChunk * 2, b_bytes = (uint32_t)A.D * kFcKChunk * 2;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kBStages * stage_bytes);
  uint64_t* empty = full + kBStages;
  uint64_t* bar_acc = empty + kBStages;
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(bar_acc + 1);
  if (tid == 0) {
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(bar_acc, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_rt(tmem_s, A.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_s;
  const int nchunks = A.K / kFcKChunk;
  const uint8_t* a_src = A.feat + tile * ((int64_t)A.K * 256);
  if (tid == 0) {
    auto issue = [&](int c) {
      const int s = c % kBStages;
      if (c >= kBStages) mbar_wait(&empty[s], (uint32_t)(((c / kBStages) - 1) & 1));
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      bulk_g2s(stages + (size_t)s * stage_bytes, a_src + (size_t)c * a_bytes, a_bytes, &full[s]);
      bulk_g2s(stages + (size_t)s * stage_bytes + a_bytes, A.wpack + (size_t)c * b_bytes, b_bytes,
               &full[s]);
    };
    int issued = 0;
    for (; issued < kBStages - 1 && issued < nchunks; ++issued) issue(issued);
    const uint32_t idesc = idesc_bf16_f32(128, A.D);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kBStages;
      mbar_wait(&full[s], (uint32_t)((c / kBStages) & 1));
      tc_fence_after();
      const uint32_t as = smem_u32(stages + (size_t)s * stage_bytes), bs = as + a_bytes;
#pragma unroll
      for (int kk = 0; kk < kFcKChunk / 16; ++kk)
        umma_bf16(tmem, sdesc(as + kk * 2 * 2048, 2048, 128),
                  sdesc(bs + kk * 2 * A.D * 16, A.D * 16, 128), idesc, (c > 0 || kk > 0) ? 1u : 0u);
      umma_commit(&empty[s]);
      if (issued < nchunks) issue(issued++);
    }
    umma_commit(bar_acc);
  }
  __syncwarp();
  mbar_wait(bar_acc, 0);
  tc_fence_after();
  float z = 0.0f;
  for (int cb = 0; cb < A.D / 16; ++cb) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + cb * 16, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = cb * 16 + j;
      const float h = bf2f(f2bf(fmaxf(__uint_as_float(r[j]) + A.b1[c], 0.0f)));
      z = fmaf(h, bf2f(A.w2[c]), z);
    }
  }
  z += A.b2[0];
  const int64_t row = tile * 128 + tid;
  if (row < cnt) A.logits[A.chunk_base + row] = z;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc_rt(tmem, A.tmem_cols);
}

// =================================================================== host plan
struct LayerPlan {
  int cin, cout, hin, hp, wp, hpool;
  int n_tiles, n_pass, pass_n, mma_n, chunk_ch, chunks_per_pass, chunk_bytes, plane_rows;
  uint32_t tmem_cols;
  size_t smem;
  size_t w_off, w_bytes;
  size_t in_off;
  int64_t in_frame_bytes;
};
struct CnnPlan {
  int L, C, D, K, hfinal;
  size_t w1_off, w1_bytes;
  LayerPlan lay[4];        // lay[1..L-1] = shifted-window layers
  size_t fc_off, fc_bytes;
  size_t act2_off;
  int64_t act2_frame_bytes;
  size_t feat_off;
  size_t total;
  int64_t chunk;
};

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static bool make_plan(const noscope_cnn_arch& a, int64_t n_max, CnnPlan* P) {
  CnnPlan p{};
  p.L = a.n_conv;
  p.C = a.base_filters;
  p.D = a.dense;
  p.chunk = std::min<int64_t>(kCnnChunk, std::max<int64_t>(128, (n_max + 127) / 128 * 128));
  size_t off = 256;  // status words etc. live before the CNN region (caller offset)
  p.w1_off = off;
  p.w1_bytes = (size_t)p.C * 32 * 2;  // [4 kc][C][8]: K = 27 padded to 32
  off = align_up(off + p.w1_bytes, 256);
  int h = 25, cin = p.C;
  for (int l = 1; l < p.L; ++l) {
    LayerPlan& L = p.lay[l];
    L.cin = cin;
    L.cout = cin * 2;
    L.hin = h;
    L.hp = h + 2;
    L.wp = h + 2;
    L.hpool = h / 2;
    const int rows = 2 * L.hpool * L.wp;
    L.n_tiles = (rows + 127) / 128;
    int pn = std::min(L.cout, 512);
    while (L.n_tiles * pn > 512) pn /= 2;
    L.pass_n = pn;
    L.n_pass = L.cout / pn;
    L.mma_n = std::min(pn, 256);
    int cc = L.cin;
    while ((size_t)L.pass_n * cc * 2 > 32768) cc /= 2;
    L.chunk_ch = cc;
    L.chunks_per_pass = 9 * L.cin / cc;
    L.chunk_bytes = L.pass_n * cc * 2;
    L.plane_rows = L.n_tiles * 128 + 2 * L.wp + 2;
    L.tmem_cols = 32;
    while ((int)L.tmem_cols < L.n_tiles * L.pass_n) L.tmem_cols <<= 1;
    L.in_frame_bytes = (int64_t)(L.cin / 8) * L.hp * L.wp * 16;
    L.w_off = off;
    L.w_bytes = (size_t)L.cout * 9 * L.cin * 2;
    off = align_up(off + L.w_bytes, 256);
    size_t sm = align_up((size_t)(L.cin / 8) * L.plane_rows * 16, 1024);
    sm += (size_t)kBStages * L.chunk_bytes;
    sm += (size_t)L.n_tiles * 128 * kEpCols * 2;
    sm += (2 * kBStages + 2) * 8 + 16;
    L.smem = sm + 1024;
    if (L.smem > 227 * 1024) return false;
    cin = L.cout;
    h = L.hpool;
  }
  p.hfinal = h;
  p.K = h * h * cin;
  if (p.K % kFcKChunk) return false;
  p.fc_off = off;
  p.fc_bytes = (size_t)p.D * p.K * 2;
  off = align_up(off + p.fc_bytes, 256);
  // activations for one chunk of frames
  p.act2_frame_bytes = (int64_t)(p.C / 8) * 27 * 27 * 16;
  p.act2_off = off;
  off = align_up(off + (size_t)p.chunk * p.act2_frame_bytes, 1024);
  for (int l = 2; l < p.L; ++l) {
    p.lay[l].in_off = off;
    off = align_up(off + (size_t)p.chunk * p.lay[l].in_frame_bytes, 1024);
  }
  p.lay[1].in_off = p.act2_off;
  p.feat_off = off;
  off = align_up(off + (size_t)p.chunk * p.K * 2, 1024);
  p.total = off;
  *P = p;
  return true;
}

bool cnn_arch_supported(const noscope_cnn_arch& a) {
  if (a.in_w != 50 || a.in_h != 50) return false;
  if (a.n_conv != 2 && a.n_conv != 4) return false;
  if (a.base_filters != 32 && a.base_filters != 64) return false;
  if (a.dense != 32 && a.dense != 64 && a.dense != 128 && a.dense != 256) return false;
  CnnPlan p;
  return make_plan(a, 128, &p);
}

size_t cnn_ws_bytes(const noscope_cnn_arch& a, int64_t n_max) {
  CnnPlan p;
  if (!make_plan(a, n_max, &p)) return 0;
  return p.total;
}

// Debug/test helper: offsets of the internal activation buffers (see noscope_api.cu).
bool cnn_debug_layout(const noscope_cnn_arch& a, int64_t n_max, int64_t* out) {
  CnnPlan p;
  if (!make_plan(a, n_max, &p)) return false;
  out[0] = (int64_t)p.act2_off;
  out[1] = p.act2_frame_bytes;
  for (int l = 2; l < 4; ++l) {
    out[2 * l - 2] = l < p.L ? (int64_t)p.lay[l].in_off : -1;
    out[2 * l - 1] = l < p.L ? p.lay[l].in_frame_bytes : 0;
  }
  out[6] = (int64_t)p.feat_off;
  out[7] = p.K;
  out[8] = p.chunk;
  return true;
}

static void pack(const uint16_t* w, int rows, int Kreal, int Kpad, int pn, uint8_t* out,
                 cudaStream_t st) {
  int64_t total = (int64_t)rows * Kpad;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 4 * kNumSMs);
  pack_kernel<<<grid, 256, 0, st>>>(w, rows, Kreal, Kpad, pn, reinterpret_cast<uint16_t*>(out));
  count_launch();
}

noscope_status launch_cnn(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                          const uint8_t* small, int64_t small_pitch, const int32_t* idx,
                          const int64_t* n_dev, int64_t n_max, float* logits, void* ws_v,
                          uint32_t* status, cudaStream_t st) {
  (void)status;
  CnnPlan P;
  if (!make_plan(a, n_max, &P)) return NOSCOPE_INVALID_ARGUMENT;
  if (n_max <= 0) return NOSCOPE_OK;
  uint8_t* ws = reinterpret_cast<uint8_t*>(ws_v);
  // pack weights into the canonical UMMA layouts
  pack(w.conv_w[0], P.C, 27, 32, P.C, ws + P.w1_off, st);
  if (P.C == 32) {  // fused path: bias folded into K columns 27/28 of conv1
    noscope_status sb = pack_conv12_bias(w.conv_b[0], ws + P.w1_off, st);
    if (sb != NOSCOPE_OK) return sb;
  }
  for (int l = 1; l < P.L; ++l) {
    const LayerPlan& L = P.lay[l];
    pack(w.conv_w[l], L.cout, 9 * L.cin, 9 * L.cin, L.pass_n, ws + L.w_off, st);
  }
  pack(w.fc1_w, P.D, P.K, P.K, P.D, ws + P.fc_off, st);
  NS_LAUNCH_CHECK();

  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(convN_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(fc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(conv1_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(conv1_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    attr = true;
  }
  const bool fused12 = P.C == 32;  // conv1+conv2 in one kernel (cnn_fused.cu)
  for (int64_t base = 0; base < n_max; base += P.chunk) {
    const int64_t len = std::min<int64_t>(P.chunk, n_max - base);
    if (fused12) {
      FusedArgs fa{};
      fa.small = small;
      fa.small_pitch = small_pitch;
      fa.idx = idx;
      fa.n_dev = n_dev;
      fa.n_max = n_max;
      fa.chunk_base = base;
      fa.chunk_len = len;
      fa.w1 = ws + P.w1_off;
      fa.w2 = ws + P.lay[1].w_off;
      fa.b1 = w.conv_b[0];
      fa.b2 = w.conv_b[1];
      fa.mean[0] = a.chan_mean[0];
      fa.mean[1] = a.chan_mean[1];
      fa.mean[2] = a.chan_mean[2];
      fa.to_features = P.L == 2 ? 1 : 0;
      fa.out = P.L == 2 ? ws + P.feat_off : ws + P.lay[2].in_off;
      fa.K_feat = P.K;
      fa.out_frame_bytes = P.L == 2 ? 0 : P.lay[2].in_frame_bytes;
      noscope_status s = launch_conv12_fused(fa, (int)std::min<int64_t>(len, kNumSMs), st);
      if (s != NOSCOPE_OK) return s;
    }
    Conv1Args c1{};
    c1.small = small;
    c1.small_pitch = small_pitch;
    c1.idx = idx;
    c1.n_dev = n_dev;
    c1.n_max = n_max;
    c1.chunk_base = base;
    c1.chunk_len = len;
    c1.wpack = reinterpret_cast<const uint16_t*>(ws + P.w1_off);
    c1.bias = w.conv_b[0];
    c1.mean[0] = a.chan_mean[0];
    c1.mean[1] = a.chan_mean[1];
    c1.mean[2] = a.chan_mean[2];
    c1.act_out = ws + P.act2_off;
    c1.out_frame_bytes = P.act2_frame_bytes;
    const int g1 = (int)std::min<int64_t>(len, 3 * kNumSMs);
    if (!fused12) {
      conv1_kernel<64><<<g1, kCnnThreads, conv1_smem_bytes<64>(), st>>>(c1);
      NS_LAUNCH_CHECK();
      count_launch();
    }
    for (int l = fused12 ? 2 : 1; l < P.L; ++l) {
      const LayerPlan& L = P.lay[l];
      ConvNArgs c{};
      c.act_in = ws + L.in_off;
      c.in_frame_bytes = L.in_frame_bytes;
      c.cin = L.cin;
      c.hp = L.hp;
      c.wp = L.wp;
      c.last = (l == P.L - 1);
      if (!c.last) {
        c.act_out = ws + P.lay[l + 1].in_off;
        c.out_frame_bytes = P.lay[l + 1].in_frame_bytes;
        c.hp_out = P.lay[l + 1].hp;
        c.wp_out = P.lay[l + 1].wp;
      }
      c.feat = ws + P.feat_off;
      c.K_feat = P.K;
      c.wpack = ws + L.w_off;
      c.bias = w.conv_b[l];
      c.cout = L.cout;
      c.hpool = L.hpool;
      c.n_tiles = L.n_tiles;
      c.n_pass = L.n_pass;
      c.pass_n = L.pass_n;
      c.mma_n = L.mma_n;
      c.chunk_ch = L.chunk_ch;
      c.chunks_per_pass = L.chunks_per_pass;
      c.chunk_bytes = L.chunk_bytes;
      c.plane_rows = L.plane_rows;
      c.tmem_cols = L.tmem_cols;
      c.n_dev = n_dev;
      c.n_max = n_max;
      c.chunk_base = base;
      c.chunk_len = len;
      const int g = (int)std::min<int64_t>(len, kNumSMs);
      convN_kernel<<<g, kCnnThreads, L.smem, st>>>(c);
      NS_LAUNCH_CHECK();
      count_launch();
    }
    FcArgs f{};
    f.feat = ws + P.feat_off;
    f.K = P.K;
    f.D = P.D;
    f.wpack = ws + P.fc_off;
    f.b1 = w.fc1_b;
    f.w2 = w.fc2_w;
    f.b2 = w.fc2_b;
    f.logits = logits;
    f.n_dev = n_dev;
    f.n_max = n_max;
    f.chunk_base = base;
    f.chunk_len = len;
    f.tmem_cols = tmem_cols_host(P.D);
    const size_t fsm = (size_t)kBStages * (128 * kFcKChunk * 2 + P.D * kFcKChunk * 2) +
                       (2 * kBStages + 1) * 8 + 16 + 1024;
    fc_kernel<<<(int)((len + 127) / 128), kCnnThreads, fsm, st>>>(f);
    NS_LAUNCH_CHECK();
    count_launch();
  }
  return NOSCOPE_OK;
}

}  // namespace ns
