// internal.h — host/device declarations shared by the NoScope CUDA sources.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/noscope.h"

namespace ns {

constexpr int kMaxGrid = 16;      // blocked-DD grid side limit (g*g <= 256 blocks)
constexpr int kMaxOutW = 53;      // out_w*3 <= 160 box-mean threads own one output column each
constexpr int kMaxBox = 2048;     // max source pixels per output pixel (exact magic division)

// Optional stage timing (noscope_cascade_run_profiled) and launch counting.
struct Prof {
  cudaEvent_t ev[16];
  int n;
};
inline void prof_mark(Prof* p, cudaStream_t st) {
  if (p && p->n < 16) cudaEventRecord(p->ev[p->n++], st);
}
uint64_t& launch_counter();  // kernels launched by the calling host thread

// Per-device caches.  Function attributes and occupancy belong to a device
// context, so a process that drives several GPUs (cudaSetDevice between calls)
// needs them once per device, keyed by the current device ordinal.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  return cudaGetDevice(&d) == cudaSuccess && d >= 0 && d < kMaxDevices ? d : 0;
}
struct DeviceOnce {           // first() is true once per device
  std::atomic<bool> done[kMaxDevices]{};
  bool first() { return !done[current_device()].exchange(true); }
};
struct DeviceInt {            // an int cached per device (0 = not yet known)
  std::atomic<int> v[kMaxDevices]{};
  int get() { return v[current_device()].load(); }
  void set(int x) { v[current_device()].store(x); }
};
inline void count_launch(int k = 1) { launch_counter() += (uint64_t)k; }

struct DsGeom {
  int out_w, out_h, metric, grid;
  const float* lr_w;
  float lr_b;
  double delta;
};

// Frames that must be downsampled: checked frames (tau % t_skip == 0) and,
// in mode 1, anchors of checked frames ((tau + k) % t_skip == 0).  Ordinals
// m enumerate them in tau order: tau = (m / nres) * t_skip + res[m % nres].
struct NeededSet {
  int64_t m0, m1, tau0;
  int t_skip, nres;
  int res[2];
  __host__ __device__ int64_t frame_of(int64_t m) const {
    int64_t p = m / nres;
    return p * t_skip + res[m - p * nres] - tau0;
  }
};

inline int64_t needed_count(const NeededSet& s, int64_t x) {  // # needed tau in [0, x)
  int64_t c = 0;
  for (int r = 0; r < s.nres; ++r)
    if (x > s.res[r]) c += (x - s.res[r] + s.t_skip - 1) / s.t_skip;
  return c;
}

inline NeededSet make_needed_set(const noscope_dd_config& cfg, int64_t tau0, int64_t n) {
  NeededSet s{};
  s.t_skip = cfg.t_skip_frames;
  s.tau0 = tau0;
  s.res[0] = 0;
  s.nres = 1;
  if (cfg.mode == 1) {
    int r = (int)((s.t_skip - (cfg.t_diff_frames % s.t_skip)) % s.t_skip);
    if (r != 0) {
      s.res[1] = r;
      s.nres = 2;
    }
  }
  s.m0 = needed_count(s, tau0);
  s.m1 = needed_count(s, tau0 + n);
  return s;
}

inline int64_t small_bytes_of(const noscope_dd_config& c) { return (int64_t)c.out_w * c.out_h * 3; }
inline int64_t state_ring_pitch(const noscope_dd_config& c) { return (small_bytes_of(c) + 15) & ~15ll; }
inline int64_t state_ring_bytes(const noscope_dd_config& c) {
  return c.mode == 1 ? (int64_t)c.t_diff_frames * state_ring_pitch(c) : 0;
}
inline int state_label_len(const noscope_dd_config& c) {
  const int ts = c.t_skip_frames;
  if (c.mode != 1) return ts;
  const int K = (c.t_diff_frames + ts - 1) / ts;
  return (K + 1) * ts;
}

// ---- launchers (all asynchronous on `st`)
// Fired-frame queue of the overlapped cascade (noscope_api.cu): dd_kernel's scorer
// appends every frame it fires (reserve a slot with an atomic, then publish the frame
// index with a release store after its small frame is written); the queue-mode CNN
// (cnn_fused.cu) claims slots and reads the frames while the DD is still streaming.
struct FiredQueue {
  int32_t* q;                   // [n] frame indices (call-relative), -1 until published
  unsigned long long* count;    // slots reserved by dd_kernel
  unsigned long long* claim;    // slots claimed by CNN CTAs
  unsigned* done;               // dd_kernel CTAs finished (all entries published)
  int producers;                // dd_kernel grid size (0 until launched)
};
constexpr size_t kFqHeaderBytes = 256;   // count @0, claim @8, done @16
// fq (nullable): also append fired frames to the queue (dd_kernel path only; the
// identity kernel does not produce a queue: fq->producers stays 0).  reserve_sms:
// SMs left free for a concurrently running kernel.
noscope_status launch_diff_detect(const noscope_dd_config& cfg, const uint8_t* frames,
                                  const noscope_frames_desc& desc, int64_t n, int64_t tau0,
                                  uint8_t* state, uint8_t* small, int64_t small_pitch,
                                  double* score, uint8_t* disp, uint32_t* status,
                                  unsigned* flags, cudaStream_t st, Prof* prof = nullptr,
                                  FiredQueue* fq = nullptr, int reserve_sms = 0);
// Would launch_diff_detect use the band-pipeline dd_kernel (and so feed a queue)?
bool dd_uses_band_kernel(const noscope_dd_config& cfg, const noscope_frames_desc& desc);
// fp32-accurate tcgen05 GEMM (gemm_tc.cu, 3xTF32): C[m][n] = sum_k A(m,k) B(k,n)
// with A(m,k) = A[m*sam + k*sak], B(k,n) = B[n*sbn + k*sbk]; `part` = split-K
// scratch of tc_gemm_part_floats(M, N, K) floats (nullable when that is 0).
struct TcGemmArgs {
  const float* A;
  int64_t sam, sak;
  const float* B;
  int64_t sbn, sbk;
  float* C;
  int64_t ldc;
  int M, N;
  int64_t K;
  int ksplit;
  int64_t kper;
  float* part;
};
size_t tc_gemm_part_floats(int M, int N, int64_t K);
noscope_status tc_gemm(const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn, int64_t sbk, float* C,
                       int64_t ldc, int M, int N, int64_t K, float* part, cudaStream_t st);

// Whether dd_kernel's band ring (>= 2 stages of one output row's source rows per
// worker group, at least one group) fits shared memory for this source size.
bool dd_frames_fit(const noscope_dd_config& cfg, const noscope_frames_desc& desc);
size_t dd_flags_bytes();  // workspace for the per-CTA completion flags
noscope_status launch_state_update(const noscope_dd_config& cfg, const uint8_t* small,
                                   int64_t small_pitch, uint8_t* state, int64_t tau0, int64_t n,
                                   const uint8_t* labels, cudaStream_t st);

// Stable compaction of fired frames (+ fills skipped frames' disposition/score).
size_t compact_ws_bytes(int64_t n);
// pos_pf (nullable): per-frame position in idx_out, written for the selected frames.
noscope_status launch_compact_fired(const uint8_t* disp_in, uint8_t* disp, double* score,
                                    int64_t n, int64_t tau0, int t_skip, int32_t* idx_out,
                                    int64_t* count_out, void* scan_ws, cudaStream_t st,
                                    int32_t* pos_pf = nullptr);
// Routing of compacted logits + compaction of uncertain ones.
noscope_status launch_route(noscope_route r, const float* logits, const int64_t* n_dev,
                            int64_t n_max, const int32_t* frame_idx, uint8_t* route_out,
                            uint8_t* route_pf, int32_t* unc_out, int64_t* n_unc,
                            int32_t* unc_pos_pf, float* logits_pf, uint64_t* counters,
                            void* scan_ws, uint32_t* status, cudaStream_t st);
// Label resolution for one chunk.
size_t labels_ws_bytes(int64_t n);
noscope_status launch_labels(const noscope_dd_config& cfg, int64_t tau0, int64_t n,
                             const uint8_t* disp, const uint8_t* route_pf,
                             const int32_t* unc_pos_pf, const uint8_t* answers,
                             const uint8_t* lab_hist, uint8_t* labels, uint8_t* route_out,
                             void* lws, cudaStream_t st);

// Specialized CNN.
// Fused conv1+conv2 (base_filters = 32), cnn_fused.cu.
struct FusedArgs {
  int C1;              // conv1 channels: 32 (conv2 fused) or 16 / 64 (conv1 only -> stacked map)
  const uint8_t* small;
  int64_t small_pitch;
  const int32_t* idx;
  const int64_t* n_dev;
  int64_t n_max, chunk_base, chunk_len;
  const uint8_t* w1;   // packed [4][C1][8]
  const uint8_t* w2;   // packed [36][64][8]
  const float* b1;
  const float* b2;
  float mean[3];
  int to_features;     // 1: FC feature tiles, 0: stacked map (next layer's input)
  uint8_t* out;
  int K_feat;          // feature length (to_features)
  int64_t out_rows;    // rows per channel-group plane of the stacked map (!to_features)
  // queue mode (conv2-fused variants writing FC features): frames are claimed from a
  // FiredQueue instead of idx/n_dev; the features of queue slot p go to row p.
  //   qmode 1 ("side"): runs beside dd_kernel, claims published slots until every
  //           dd_kernel CTA is done, then stops (the rest is left to qmode 2);
  //   qmode 2 ("tail"): launched after dd_kernel, claims every remaining slot.
  int qmode;           // 0 = index mode
  FiredQueue fq;
  long long* dbg;      // experiments only (NS_EXP & 256 builds): per-warp wait cycles
};
size_t conv12_fused_smem();

// Generic conv layer (cnn_gemm.cu): batched implicit GEMM over the "stacked"
// activation layout.  A map of H x W pixels x Cin channels for a chunk of F
// frames is stored as Cin/8 planes [cg][R rows][8 ch] (bf16, 16 B per row):
//   row(f, y, x) = G + f*P + (y + 1)*Wq + x,  Wq = W + 1, P = (H + 1)*Wq, G = Wq + 1,
// with every other row zero: one zero row above each frame and one zero column
// right of each row are the 3x3 conv's zero padding on all four sides (the
// column right of row y-1 is the left neighbour of row y).
struct ConvGGeom {
  int tiled;                 // 1: 2-D tile variant (cnn_tile.cu), even row period H + 1
  int cin_real, cin_eff, cout, H, W;   // cin_eff = cin_real (multiple of 16)
  int N, passes, steps;      // MMA N (<= 256) per pass over Cout; K16 steps
  int MT, nacc, nA, bstages; // M tiles per unit, accumulator sets, A / B ring depths
  int kb;                    // K16 steps per B ring stage
  int S, rows_blk;           // unit stride in rows; rows loaded per unit per plane
  int64_t R;                 // rows per plane of the layer input (chunk)
  uint32_t tmem_cols;
  size_t oB, oStage, oWin, oBias, oBar, smem;
};
bool make_convg_geom(int cin_real, int cout, int H, int64_t chunk, ConvGGeom* g);
inline int64_t sl_rows(int H, int W, int64_t frames, int64_t slack) {
  const int64_t Wq = W + 1;
  return (Wq + 1) + frames * (H + 1) * Wq + slack;
}
struct ConvGArgs {
  ConvGGeom g;
  const uint8_t* in;       // stacked input planes
  const uint8_t* wpack;    // [passes][steps][2][N][8] bf16
  const float* bias;
  int to_features;
  uint8_t* out;            // stacked output planes (R_out rows) or FC feature tiles
  int64_t out_rows;
  int K_feat;
  const int64_t* n_dev;
  int64_t n_max, chunk_base, chunk_len;
  long long* dbg;          // experiments only (NS_EXP & 256 builds)
};
noscope_status launch_convg(const ConvGArgs& a, cudaStream_t st);
bool make_convt_geom(int cin, int cout, int H, int64_t chunk, ConvGGeom* g);
noscope_status launch_convt(const ConvGArgs& a, cudaStream_t st);
noscope_status pack_convg(const uint16_t* w, const ConvGGeom& g, uint8_t* out, cudaStream_t st);
noscope_status launch_conv12_fused(const FusedArgs& a, int grid, cudaStream_t st);
size_t cnn_ws_bytes(const noscope_cnn_arch& a, int64_t n_max);
noscope_status launch_cnn(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                          const uint8_t* small, int64_t small_pitch, const int32_t* idx,
                          const int64_t* n_dev, int64_t n_max, float* logits, void* ws,
                          uint32_t* status, cudaStream_t st);
// Queue mode of the specialized CNN (the overlapped cascade, noscope_api.cu): archs
// whose conv1+conv2 kernel writes the FC features (conv2 fused, L = 2).  The
// workspace holds the features of up to n_max queue slots (no 32,768-frame chunks).
bool cnn_queue_supported(const noscope_cnn_arch& a);
size_t cnn_queue_ws_bytes(const noscope_cnn_arch& a, int64_t n_max);
noscope_status cnn_queue_pack(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                              int64_t n_max, void* ws, cudaStream_t st);
noscope_status cnn_queue_conv(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                              const uint8_t* small, int64_t small_pitch, const FiredQueue& fq,
                              int qmode, int grid, int64_t n_max, void* ws, cudaStream_t st);
// FC over queue slots [0, *fq.count): logit of slot p -> logits[pos_pf[fq.q[p]]].
noscope_status cnn_queue_fc(const noscope_cnn_arch& a, const noscope_cnn_weights& w,
                            const FiredQueue& fq, int64_t n_max, const int32_t* pos_pf,
                            float* logits, void* ws, cudaStream_t st);

// DD fitting (fit.cu).
size_t fit_ws_bytes(int64_t n, int32_t d, int64_t small_bytes);
noscope_status launch_reference_image(const uint8_t* small, int64_t pitch, int bytes, const uint8_t* labels,
                                      int64_t n, uint8_t* ref, void* ws, uint64_t* neg_count_host,
                                      cudaStream_t st);
noscope_status launch_block_features(const noscope_dd_config& c, const uint8_t* small, int64_t pitch,
                                     int64_t n, double* feats, cudaStream_t st);
noscope_status launch_lr_fit(const double* F, const uint8_t* t, int64_t n, int d, int max_iters, double tol,
                             double l2, double* wb_host, double* info_host, void* ws, cudaStream_t st);

// CBO search helper (cbo.cu).
noscope_status launch_records_a(const double* score, const uint8_t* y, int64_t n, int mode, int k,
                                int t_skip, uint8_t* a, cudaStream_t st);

noscope_status launch_eval_labels(const uint8_t* pred, const uint8_t* ref, int64_t n, int window,
                                  int agree_min, unsigned long long* counters, int64_t* out_host,
                                  cudaStream_t st);

// Specialized-CNN training (train.cu).
int64_t train_param_count(const noscope_cnn_arch& a);
size_t train_ws_bytes(const noscope_cnn_arch& a, int batch);
noscope_status launch_cnn_train(const noscope_cnn_arch& a, const noscope_train_config& cfg, float* P,
                                const uint8_t* small, int64_t pitch, const uint8_t* labels, const int32_t* perms,
                                int64_t n_train, const int32_t* val_idx, int64_t n_val, double* hist,
                                int32_t* epochs_run, void* ws, cudaStream_t st);
noscope_status launch_params_to_weights(const noscope_cnn_arch& a, const float* P, const noscope_cnn_weights& wt,
                                        cudaStream_t st);

// Threshold sweep.
size_t sweep_ws_bytes(int32_t n_delta, int32_t m);
noscope_status launch_sweep(int32_t phase, const double* s, const float* z, const uint8_t* y,
                            const uint8_t* a, int64_t n, const double* delta, int32_t nd,
                            const float* u, int32_t m, uint64_t* hist, const noscope_timing& t,
                            uint64_t fp_limit, uint64_t fn_limit,
                            const noscope_sweep_tables* tables, noscope_sweep_best* best_host,
                            void* ws, cudaStream_t st, bool* infeasible);

}  // namespace ns
