/*
 * noscope.h — C ABI of the B200-native NoScope cascade hot path.
 *
 * NoScope (Kang et al., "NoScope: Optimizing Neural Network Queries over Video
 * at Scale", arXiv 1703.02529; text at /root/reference/PAPER.md, cited P:<line>)
 * answers a binary per-frame query ("is an object of class X visible?") by
 * reproducing a reference network's decisions through a cascade: frame
 * skipping and a difference detector, a specialized CNN with two
 * confidence thresholds c_low / c_high, and the reference network
 * only for the uncertain frames; a cost-based optimizer sweeps the thresholds
 * (delta_diff, c_low, c_high) under FP/FN targets.
 *
 * This library exports that hot path as four calls (BASELINE.json north_star):
 *   noscope_diff_detect        downsample + difference detector + compaction
 *   noscope_specialized_infer  the specialized CNN on compacted frames
 *   noscope_cascade_run        the whole per-frame cascade on one chunk
 *   noscope_threshold_sweep    the CBO's (delta_diff, c_low, c_high) sweep
 * plus small helpers (size queries, state init, routing, status strings).
 *
 * Conventions (all entry points)
 *  - Pointers named *_dev / frames / small / ws / state are DEVICE pointers
 *    (any CUDA allocation visible to the current device, e.g. the PyTorch
 *    caching allocator); *_host pointers are host memory.  The caller owns
 *    every buffer; the library never allocates or frees device memory and
 *    holds no global state beyond per-device caches of kernel attributes, so
 *    calls on different streams with distinct workspaces/states are
 *    independent.  Two calls create short-lived CUDA objects of their own:
 *    noscope_cnn_train captures and replays a CUDA graph of one training step
 *    on a private stream, and the opt-in overlapped schedule of
 *    noscope_cascade_run (NOSCOPE_OVERLAP=1) uses a private side stream and two
 *    events; all are destroyed before the call returns.
 *  - Work is enqueued asynchronously on `stream` (a cudaStream_t; 0 = legacy
 *    default stream).  Exceptions: noscope_threshold_sweep with phase 2/3 and
 *    any call given a non-null *_host output synchronise `stream` once to copy
 *    the result back.
 *  - Host-side validation happens before any launch and returns
 *    NOSCOPE_INVALID_ARGUMENT / NOSCOPE_SHAPE / NOSCOPE_WORKSPACE_TOO_SMALL
 *    with nothing enqueued.  Launch failures return NOSCOPE_CUDA.  Errors the
 *    device detects (NaN scores/logits) set a status word inside the workspace;
 *    noscope_check() reads it (synchronising `stream`).
 *  - Frames: uint8, row-major, channel-interleaved RGB (HWC, 3 channels);
 *    frame f starts at frames + f*frame_pitch; frame_pitch is a multiple of 16
 *    and >= round_up(width*height*3, 16).  Downsampled ("small") frames use the
 *    same convention with small_pitch.
 *  - Every device buffer must be 16-byte aligned.
 *  - Requires compute capability 10.0 (B200, sm_100a); otherwise
 *    NOSCOPE_UNSUPPORTED_DEVICE.
 */
#ifndef NOSCOPE_H_
#define NOSCOPE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* noscope_stream_t; /* == cudaStream_t */

typedef enum {
  NOSCOPE_OK = 0,
  NOSCOPE_INVALID_ARGUMENT = 1,   /* null pointer, bad enum, unsorted/duplicate candidates, lo > hi */
  NOSCOPE_SHAPE = 2,              /* downsample target > source, pitch not /16, grid > dims */
  NOSCOPE_WORKSPACE_TOO_SMALL = 3,
  NOSCOPE_CUDA = 4,               /* launch / runtime error */
  NOSCOPE_UNSUPPORTED_DEVICE = 5, /* not compute capability 10.0 */
  NOSCOPE_DATA = 6,               /* NaN score or logit detected on device */
  NOSCOPE_INFEASIBLE = 7,         /* sweep: no triple meets FP* and FN*; best-effort result written */
  NOSCOPE_LABELLER = 8            /* labeller callback returned nonzero */
} noscope_status;

const char* noscope_status_string(noscope_status s);
/* Library version, e.g. 100 = 0.1.0. */
int32_t noscope_version(void);

/* ---------------------------------------------------------------- frames */
typedef struct {
  int32_t width;        /* source W (pixels) */
  int32_t height;       /* source H (pixels) */
  int64_t frame_pitch;  /* bytes between frames, multiple of 16 */
} noscope_frames_desc;

/* ------------------------------------------------------ difference detector
 * PAPER.md §5.  Modes: "difference detection against a fixed
 * reference image ... that contains no objects" or "against an
 * earlier frame a pre-configured time t_diff seconds into the past",
 * here a fixed lag of k = t_diff_frames frames (reading R-8).  Metric: MSE over
 * the whole image, or "a blocked comparison where it subdivides each image into
 * a grid and computes the metric on every grid block" weighted by a logistic
 * regression; the blocked score is the LR logit (reading R-3).
 * A frame at unit position tau is checked iff tau % t_skip_frames == 0
 * (R-10); it fires iff score > delta_diff (strict, R-4);
 * in mode 1 the first k checked frames of a unit (tau < k) fire unconditionally.
 * Before scoring, every needed frame is downsampled by the integer box filter
 * G[i][j][c] = floor((2S + n) / 2n) over source rows [floor(iH/h), floor((i+1)H/h))
 * and columns [floor(jW/w), floor((j+1)W/w)) (reading R-1); the same
 * out_w x out_h frames feed the CNN.
 * Scores are fp64: global = (double)SSD / (double)(out_w*out_h*3) where SSD is
 * the exact integer sum of squared u8 differences; blocked: blocks of
 * floor(out/g) rows/cols (last block takes the remainder), m_k = SSD_k / n_k,
 * z = b + sum_k w_k * m_k evaluated in block order with separate fp64 rounding
 * of every product and sum (no FMA).  Skipped frames get score -inf, forced
 * fires +inf.                                                               */
typedef struct {
  int32_t mode;           /* 0 = reference image, 1 = earlier frame t-k */
  int32_t metric;         /* 0 = global MSE, 1 = blocked MSE + LR */
  int32_t out_w, out_h;   /* downsample target (<= source), e.g. 50 x 50; out_w <= 53
                             and out_w*out_h*3*255^2 < 2^32 (u32 SSDs), else
                             NOSCOPE_SHAPE */
  int32_t grid;           /* g for metric 1: 1 <= g <= min(out_w, out_h) */
  int32_t t_diff_frames;  /* k >= 1 (mode 1) */
  int32_t t_skip_frames;  /* >= 1 */
  int32_t reserved;
  double delta_diff;      /* firing threshold (MSE units, or LR logit) ; +-inf allowed */
  const uint8_t* ref_image;   /* device, out_h*out_w*3 u8 HWC (mode 0) */
  const float* lr_weights;    /* device, grid*grid fp32, row-major block order (metric 1) */
  float lr_bias;
  float reserved2;
} noscope_dd_config;

/* Disposition codes written per frame by noscope_diff_detect. */
enum { NOSCOPE_SKIPPED = 0, NOSCOPE_SUPPRESSED = 1, NOSCOPE_FIRED = 2 };

/* ------------------------------------------------------- specialized CNN
 * PAPER.md §4: shallow AlexNet-style network, "number of
 * convolutional layers (2 or 4), number of convolution units in the base layer
 * (32 or 64), and number of neurons in the dense layer", ReLU
 * hidden units, softmax output (two-class softmax == sigmoid of one logit).
 * Per layer l = 1..n_conv: 3x3 conv, stride 1, zero pad 1, Cout = base*2^(l-1)
 * ("filter doubling"), + bias, ReLU, 2x2/2 max pool (floor); flatten
 * (h, w, c); FC(dense) + bias + ReLU; FC(1) + bias -> logit z (reading R-12).
 * Input: x = bf16_RNE(clamp(((float)G - chan_mean[c]) / 127.5f, -1, 1))
 * ("mean-center the pixel values and change the dynamic range in each color
 * channel to [-1, 1]", reading R-13).  Operands bf16, accumulation
 * fp32 (tensor cores), activations rounded to bf16 after each pool / FC1.
 * Supported: n_conv in {2,4}, base_filters in {16,32,64} (the text names 32 or
 * 64, but Table 2 picks C = 16 for coral and night-street, P:1136-1140,
 * and "24 distinct configurations", = 3 C x 2 L x 4 D), dense in
 * {32,64,128,256}, in_w = in_h = 50.                                         */
typedef struct {
  int32_t n_conv, base_filters, dense, in_w, in_h;
  float chan_mean[3];
} noscope_cnn_arch;

/* Weight tensors (device).  bf16 = IEEE bfloat16 bit patterns (uint16).
 *   conv_w[l]: bf16 [Cout][3][3][Cin]      conv_b[l]: fp32 [Cout]
 *   fc1_w:     bf16 [dense][K], K = (h,w,c) of the last pooled map
 *   fc1_b:     fp32 [dense]   fc2_w: bf16 [dense]   fc2_b: fp32 [1]          */
typedef struct {
  const uint16_t* conv_w[4];
  const float* conv_b[4];
  const uint16_t* fc1_w;
  const float* fc1_b;
  const uint16_t* fc2_w;
  const float* fc2_b;
} noscope_cnn_weights;

/* ------------------------------------------------------------- routing
 * "no object" if c < c_low, "object" if c > c_high,
 * otherwise call the reference NN.  Compared on fp32 logits (c = sigmoid(z));
 * equality defers to the reference (reading R-5); lo <= hi; +-inf allowed.  */
typedef struct {
  float lo_logit;   /* logit(c_low)  */
  float hi_logit;   /* logit(c_high) */
} noscope_route;

/* Per-frame route codes written by noscope_cascade_run / noscope_route_logits. */
enum { NOSCOPE_R_SKIP = 0, NOSCOPE_R_SUPP = 1, NOSCOPE_R_NEG = 2, NOSCOPE_R_POS = 3, NOSCOPE_R_UNC = 4 };

/* Reference-network stand-in.  Called once per cascade chunk on the
 * uncertain frames: idx_dev[i] (i < *n_dev, device count, <= n_max) are chunk
 * frame indices; the callee writes answers_dev[i] in {0,1} for frame
 * frame_index_base + idx_dev[i], enqueued on `stream`.  Return 0 on success. */
typedef int (*noscope_labeller_fn)(void* user, const int32_t* idx_dev, const int64_t* n_dev,
                                   int64_t n_max, int64_t frame_index_base,
                                   uint8_t* answers_dev, noscope_stream_t stream);

typedef struct {
  int64_t n_frames, n_skipped, n_suppressed, n_fired, n_neg, n_pos, n_uncertain;
} noscope_run_stats;

/* ------------------------------------------------------------ size queries */
typedef enum {
  NOSCOPE_OP_DIFF_DETECT = 0,
  NOSCOPE_OP_SPECIALIZED_INFER = 1,
  NOSCOPE_OP_CASCADE_RUN = 2,
  NOSCOPE_OP_THRESHOLD_SWEEP = 3
} noscope_op;

/* Workspace bytes for `op` on up to n_frames frames (sweep: n_delta, m
 * candidates; other ops ignore them).  arch may be null for ops without the
 * CNN; dd may be null for ops without the detector.  0 on invalid input.  */
size_t noscope_workspace_bytes(noscope_op op, const noscope_dd_config* dd,
                               const noscope_cnn_arch* arch, int64_t n_frames,
                               int32_t n_delta, int32_t m);

/* Per-stream carried state for chunked processing of one unit: the last k
 * downsampled frames (mode 1 anchors across chunk boundaries) and the last
 * max(k, t_skip) emitted labels.  Device memory, caller-owned.               */
size_t noscope_stream_state_bytes(const noscope_dd_config* dd);
/* Zeroes the state (call once per unit before its first chunk). */
noscope_status noscope_stream_state_init(const noscope_dd_config* dd, void* state_dev,
                                         noscope_stream_t stream);

/* ---------------------------------------------------------- entry points */

/* Downsample + difference detector + stable compaction over frames
 * [seg_offset, seg_offset + n_frames) of one unit.
 *  frames:        device, n_frames frames described by `desc`.
 *  seg_offset:    tau of frames[0] within its unit (>= 0).
 *  stream_state:  nullable; if non-null it supplies the anchors of frames whose
 *                 t-k lies before seg_offset (mode 1) and is updated with this
 *                 chunk's last frames.  Required in mode 1 when seg_offset > 0.
 *  small_out:     device [n_frames][small_pitch] u8; rows of frames that are
 *                 neither checked nor a future anchor are left unwritten.
 *  score_out:     device fp64 [n_frames] (nullable).
 *  disposition_out: device u8 [n_frames] NOSCOPE_SKIPPED/SUPPRESSED/FIRED.
 *  fired_idx_out: device i32 [n_frames] (nullable): ascending indices (into
 *                 this chunk) of fired frames; n_fired_dev: device i64 count.
 *  Errors: NOSCOPE_SHAPE if out_w > width or out_h > height, pitches not /16,
 *  out_w > 53, out_w*out_h*3*255^2 >= 2^32, a box taller than 257 rows or
 *  larger than 2,048 pixels, or one output row's source rows ("band",
 *  box_h*width*3 bytes) too large for a 2-stage shared-memory ring (about
 *  110 KB: every source size in PAPER.md Table 1, up to 1170x1080 -> 50x50,
 *  is accepted; 1920x1080 -> 50x50 is not).                                  */
noscope_status noscope_diff_detect(const noscope_dd_config* dd, const uint8_t* frames,
                                   noscope_frames_desc desc, int64_t n_frames,
                                   int64_t seg_offset, void* stream_state,
                                   uint8_t* small_out, int64_t small_pitch, double* score_out,
                                   uint8_t* disposition_out, int32_t* fired_idx_out,
                                   int64_t* n_fired_dev, void* ws, size_t ws_bytes,
                                   noscope_stream_t stream);

/* Specialized CNN logits for frames small[idx[i]] (i < n).
 *  small_frames: device u8 [*][small_pitch], each in_h x in_w x 3.
 *  idx:          device i32 (nullable: dense 0..n-1).
 *  n_dev:        device i64 count (nullable: n = n_max); must be <= n_max.
 *  logits_out:   device fp32 [n_max]; entries >= n are left unwritten.      */
noscope_status noscope_specialized_infer(const noscope_cnn_arch* arch,
                                         const noscope_cnn_weights* weights,
                                         const uint8_t* small_frames, int64_t small_pitch,
                                         const int32_t* idx, const int64_t* n_dev, int64_t n_max,
                                         float* logits_out, void* ws, size_t ws_bytes,
                                         noscope_stream_t stream);

/* Routing helper (step H6): route_out[i] = NEG / POS / UNC of
 * logits[i] (z < c_low -> NEG, z > c_high -> POS, else UNC; R-5) for
 * i < *n_dev (or n_max), and the stable (ascending) list of uncertain
 * positions + its count.  logits: device fp32 [n_max]; route_out: device u8
 * [n_max] (nullable); unc_idx_out: device i32 [n_max]; n_unc_dev: device i64.
 * ws: device scratch of noscope_route_workspace_bytes(n_max) bytes, 16-byte
 * aligned.  One persistent launch (classify + bitmask, grid barrier, indices).
 * Errors: NOSCOPE_INVALID_ARGUMENT for c_low > c_high or null buffers;
 * NOSCOPE_WORKSPACE_TOO_SMALL.                                              */
size_t noscope_route_workspace_bytes(int64_t n_max);
noscope_status noscope_route_logits(noscope_route r, const float* logits, const int64_t* n_dev,
                                    int64_t n_max, uint8_t* route_out, int32_t* unc_idx_out,
                                    int64_t* n_unc_dev, void* ws, size_t ws_bytes,
                                    noscope_stream_t stream);

/* Stable compaction helper (step H4, "batch input images before
 * passing them to the GPU"): idx_out[0 .. *n_out_dev) = the ascending
 * positions i < n with disposition[i] == NOSCOPE_FIRED.  Positions whose
 * tau = seg_offset + i has tau mod t_skip != 0 are first rewritten to
 * NOSCOPE_SKIPPED in place (the t_skip rule; diff_detect applies
 * the same rule before it compacts).
 *  disposition: device u8 [n] (inout); idx_out: device i32 [n];
 *  n_out_dev:   device i64.
 *  ws: device scratch of noscope_compact_workspace_bytes(n) bytes (16-byte
 *  aligned): a 1-bit-per-frame mask plus per-CTA counts.  One persistent
 *  launch: classify + mask + count, grid barrier, indices from the mask.
 *  Errors: NOSCOPE_INVALID_ARGUMENT for null buffers (n > 0), n < 0, n >= 2^31
 *  or t_skip < 1; NOSCOPE_WORKSPACE_TOO_SMALL.                               */
size_t noscope_compact_workspace_bytes(int64_t n);
noscope_status noscope_compact_fired(uint8_t* disposition, int64_t n, int64_t seg_offset,
                                     int32_t t_skip, int32_t* idx_out, int64_t* n_out_dev,
                                     void* ws, size_t ws_bytes, noscope_stream_t stream);

/* The whole cascade on one chunk of one unit:
 * diff_detect -> compaction -> specialized CNN on fired frames -> routing ->
 * labeller on uncertain frames -> per-frame labels:
 *   skipped:    label of the unit's last checked frame (tau - tau % t_skip)
 *   suppressed: 0 in mode 0 (the reference image "contains no objects",
 *               P:555); the label emitted for frame tau-k in mode 1 ("returns
 *               the same labels that it output for the previous frame")
 *   fired:      NEG -> 0, POS -> 1, UNC -> labeller answer.
 *  labels_out: device u8 [n_frames]; route_out: device u8 [n_frames] route
 *  codes (nullable); logits_out: device fp32 [n_frames] (nullable; written
 *  for fired frames only); scores_out: device fp64 [n_frames] (nullable).
 *  stream_state is required (init once per unit).  stats_host (nullable)
 *  triggers one synchronisation to copy counts back.  n_frames = 0 is a no-op
 *  (frames / labels_out may then be null; stats are all zero).
 *  Errors: NOSCOPE_INVALID_ARGUMENT for null required buffers, c_low > c_high,
 *  unaligned buffers; NOSCOPE_SHAPE as noscope_diff_detect, or a CNN input size
 *  that differs from the DD's out_w x out_h; NOSCOPE_WORKSPACE_TOO_SMALL;
 *  NOSCOPE_LABELLER if the callback returns nonzero.
 *  Schedule: serial (DD, compaction, CNN, routing, labels).  NOSCOPE_OVERLAP=1 in
 *  the environment (read per call, also by noscope_workspace_bytes, which then
 *  sizes for it) selects an overlapped schedule for chunks of >= 8,192 frames with
 *  an L = 2, C in {16, 32} CNN on source frames larger than the output: the conv
 *  kernel runs on a few SMs beside the DD, consuming fired frames as the DD
 *  publishes them.  Results are bit-identical; it is not faster on B200
 *  (DESIGN.md §9), so it is off by default.  It falls back to the serial schedule
 *  under stream capture or when the workspace was sized without it.           */
noscope_status noscope_cascade_run(const noscope_dd_config* dd, const noscope_cnn_arch* arch,
                                   const noscope_cnn_weights* weights, noscope_route route,
                                   const uint8_t* frames, noscope_frames_desc desc,
                                   int64_t n_frames, int64_t seg_offset,
                                   int64_t frame_index_base, void* stream_state,
                                   noscope_labeller_fn labeller, void* labeller_user,
                                   uint8_t* labels_out, uint8_t* route_out, float* logits_out,
                                   double* scores_out, noscope_run_stats* stats_host,
                                   void* ws, size_t ws_bytes, noscope_stream_t stream);

/* Same as noscope_cascade_run, plus device-time stage breakdown (CUDA events on
 * `stream`, synchronises once): stage_ms_host[7] = ms of 0 downsample(+mode-0
 * score) kernel, 1 mode-1 lag-score kernel, 2 compaction, 3 CNN, 4 routing,
 * 5 labeller, 6 label resolution + state update.                            */
noscope_status noscope_cascade_run_profiled(
    const noscope_dd_config* dd, const noscope_cnn_arch* arch, const noscope_cnn_weights* weights,
    noscope_route route, const uint8_t* frames, noscope_frames_desc desc, int64_t n_frames,
    int64_t seg_offset, int64_t frame_index_base, void* stream_state, noscope_labeller_fn labeller,
    void* labeller_user, uint8_t* labels_out, uint8_t* route_out, float* logits_out,
    double* scores_out, noscope_run_stats* stats_host, void* ws, size_t ws_bytes,
    noscope_stream_t stream, float* stage_ms_host);

/* Number of kernels this library has launched from the calling host thread
 * (diagnostic; used by bench.py's gpu_launches).                           */
uint64_t noscope_launch_count(void);

/* --------------------------------------------------------- threshold sweep
 * PAPER.md §6 (P:627-637 objective; P:685-701 cost model
 * E[t/frame] = f_s T_MSE + f_s f_m T_SNN + f_s f_m f_c T_Full; P:747-779 sweep).
 * Records i < n: s[i] fp64 DD score (-inf = skipped frame), z[i] fp32 CNN
 * logit, y[i] reference label, a[i] label inherited when not fired.
 * Candidates: delta_cand (n_delta, fp64, strictly ascending), logit_cand (m,
 * fp32, strictly ascending, +-inf allowed).  For each (j, l <= h):
 *   fired = s > delta_j;  FP = #(!fired & a=1 & y=0) + #(fired & z > u_h & y=0)
 *   FN = #(!fired & a=0 & y=1) + #(fired & z < u_l & y=1);  F = #fired
 *   U = #(fired & u_l <= z <= u_h);  cost = C*t_mse + F*t_snn + U*t_full (ps,
 *   C = #checked records) == N x the paper's formula;  feasible iff FP <=
 *   fp_limit and FN <= fn_limit.  best = argmin over feasible triples of
 *   (cost, U, j, -l, h); if none, NOSCOPE_INFEASIBLE and the triple minimising
 *   (max(FP-fp_limit, FN-fn_limit), cost, U, j, -l, h).
 * phase 1 ACCUMULATES the local records into `hist` (caller zeroes it first;
 * size noscope_sweep_hist_words(n_delta, m) uint64); the caller may sum `hist`
 * across GPUs (e.g. ncclAllReduce) before phase 2, which evaluates it.
 * phase 3 = 1 then 2.  phase | NOSCOPE_SWEEP_ASYNC: phase 2 enqueues the copy
 * of the best triple into best_host (page-locked memory) without synchronising
 * `stream`; the result is valid once the stream's work completes and the call
 * returns NOSCOPE_OK (read best_host->feasible for feasibility).            */
enum { NOSCOPE_SWEEP_ASYNC = 4 };
typedef struct { uint64_t t_mse_ps, t_snn_ps, t_full_ps; } noscope_timing;
typedef struct {
  int32_t j, l, h, feasible;
  uint64_t cost_ps, fp, fn, fired, uncertain, checked, total;
  double delta;
  float lo_logit, hi_logit;
} noscope_sweep_best;
/* Optional device tables (each uint64, row-major): F[n_delta], FPnf[n_delta],
 * FNnf[n_delta], FPf[n_delta][m], FNf[n_delta][m], GE[n_delta][m] =
 * #(fired & z >= u), GT[n_delta][m] = #(fired & z > u).                    */
typedef struct {
  uint64_t *F, *FPnf, *FNnf, *FPf, *FNf, *GE, *GT;
} noscope_sweep_tables;

/* The a[] column of the sweep records for one unit (tau = i; oracle
 * build_records; P:554-563 label inheritance): the label the cascade
 * would emit for record i if it were NOT fired, from the reference labels y:
 * skipped (s[i] == -inf) -> y[i - i % t_skip] (its period's checked frame);
 * checked -> 0 in mode 0 (the reference image shows no object) or y[i - k] in
 * mode 1 (0 for i < k).  s: device fp64 [n]; y, a_out: device u8 [n];
 * t_skip, k >= 1.  Asynchronous.                                              */
noscope_status noscope_sweep_records(const double* s, const uint8_t* y, int64_t n, int32_t mode, int32_t k,
                                     int32_t t_skip, uint8_t* a_out, noscope_stream_t stream);

size_t noscope_sweep_hist_words(int32_t n_delta, int32_t m);

noscope_status noscope_threshold_sweep(int32_t phase, const double* s, const float* z,
                                       const uint8_t* y, const uint8_t* a, int64_t n,
                                       const double* delta_cand, int32_t n_delta,
                                       const float* logit_cand, int32_t m, uint64_t* hist,
                                       const noscope_timing* timing, uint64_t fp_limit,
                                       uint64_t fn_limit, const noscope_sweep_tables* tables_dev,
                                       noscope_sweep_best* best_host, void* ws, size_t ws_bytes,
                                       noscope_stream_t stream);

/* ---- Difference-detector fitting -----------------
 * The configuration steps that produce the DD's inputs: the reference image of
 * mode 0 and the blocked-LR weights of metric 1.  Not on the per-frame path.
 * All three are deterministic (fixed-order reductions).                     */

/* Workspace for noscope_reference_image (small_bytes = out_w*out_h*3) and
 * noscope_lr_fit (n examples x d features); take the max of the uses.        */
size_t noscope_fit_workspace_bytes(int64_t n, int32_t d, int64_t small_bytes);

/* Reference image ("computes the reference image by averaging frames
 * where the reference model returns no labels"; SPEC build_reference_image
 * S:134-142; reading R-21): ref[p] = floor((2*S_p + m) / (2*m)) over the m
 * small frames with labels[i] == 0 (per-pixel mean rounded half up).
 * small: device, n frames of out_h*out_w*3 u8 (HWC) at small_pitch (multiple of
 * 16); labels: device u8 [n] (0 = no object); ref_out: device out_h*out_w*3 u8.
 * Synchronous (reads back m).  No negative frame -> NOSCOPE_DATA, ref_out
 * untouched (the caller falls back to the earlier-frame mode).
 * Frame bytes must not exceed 2^32/255 per CTA slice: any n is accepted.     */
noscope_status noscope_reference_image(const uint8_t* small, int64_t small_pitch, int32_t out_w,
                                       int32_t out_h, const uint8_t* labels, int64_t n,
                                       uint8_t* ref_out, void* ws, size_t ws_bytes,
                                       noscope_stream_t stream);

/* Per-frame block features (O3 blocked_mse on each frame): feats[i][k]
 * = MSE of LR block k (row-major, remainder rows/columns in the last block)
 * between small frame i and its anchor: dd->ref_image (dd->mode 0) or small
 * frame i - dd->t_diff_frames of this batch (mode 1; rows i < t_diff_frames
 * have no anchor and are NaN).  Uses dd->mode, out_w, out_h, grid (1..16),
 * t_diff_frames, ref_image; feats: device fp64 [n][grid*grid].  Asynchronous. */
noscope_status noscope_block_features(const noscope_dd_config* dd, const uint8_t* small,
                                      int64_t small_pitch, int64_t n, double* feats,
                                      noscope_stream_t stream);

/* Blocked-LR fit ("trains a logistic regression (LR) classifier to
 * weigh each block", P:850-853 (scikit-learn); SPEC train_block_weights
 * S:209-217; reading R-22): the minimiser, in fp64, of
 *   J(w, b) = mean_i [log(1 + exp(z_i)) - t_i z_i] + l2/2 |w|^2,  z_i = x_i.w + b
 * over z-scored features x (population mean/std per feature; constant
 * features std := 1).  l2 > 0 makes J strictly convex (a unique minimiser even
 * on separable data; l2 = 1/n is scikit-learn's default C = 1 per example).
 * Newton's method from w = b = 0: g = grad J; stop when max|g| <= tol;
 * H = [X 1]^T diag(p(1-p)) [X 1]/n + l2 diag(1..1, 0); Delta = -H^{-1} g
 * (Cholesky); step = the first of 1, 1/2, ..., 2^-15 meeting Armijo
 * J(v + s Delta) <= J(v) + 1e-4 s g.Delta (none: stop, the rounding floor is
 * reached); at most max_iters steps.  Reductions run in a fixed order
 * (bitwise reproducible).  Returned in raw-feature form: w_host[k] = w_k/sd_k,
 * w_host[d] = b - sum_k w_k mu_k / sd_k, so the DD logit b + sum w_k m_k of
 * noscope_dd_config (lr_weights = (float)w_host[0..d), lr_bias = (float)w_host[d])
 * reproduces the fitted model.  feats: device fp64 [n][d] (finite), d <= 256;
 * targets: device u8 [n] (nonzero = 1); w_host: host fp64 [d + 1]; info_host
 * (nullable): host fp64 [4] = accepted Newton steps, max|g| at the result, J
 * at the result, stop reason (1 tol met, 2 no Armijo step, 3 max_iters).
 * Synchronous (one host sync per Newton step).
 * NOSCOPE_INVALID_ARGUMENT: l2 <= 0, tol < 0 or NaN, max_iters < 0.
 * NOSCOPE_SHAPE: d > 256.  NOSCOPE_DATA: n < 2, one class only, or a
 * non-finite feature (use the global metric).                        */
noscope_status noscope_lr_fit(const double* feats, const uint8_t* targets, int64_t n, int32_t d,
                              int32_t max_iters, double tol, double l2, double* w_host, double* info_host,
                              void* ws, size_t ws_bytes, noscope_stream_t stream);

/* ---- Full CBO search -------------------------------
 * the CBO profiles every difference detector and every specialized
 * NN on the evaluation set, sweeps (delta_diff, c_low, c_high) for each
 * combination and keeps the cheapest cascade (cost model P:696) meeting FP* /
 * FN*.  Reading R-23: every DD config and CNN runs unfiltered on all n frames
 * (one unit, tau = 0..n-1, no prior state); per (DD, CNN) pair one
 * noscope_threshold_sweep with records s = DD score, z = CNN logit, y =
 * labels, a = the label emitted when not fired (skipped -> its period's
 * checked frame's label; mode 0 -> 0; mode 1 -> label(t-k), 0 for t < k);
 * timing (t_mse_ps, that CNN's t_snn_ps, t_full_ps).  Overall argmin key:
 * (infeasible, violation, cost, U, dd index, cnn index).
 * All DD configs must have out_w = out_h = 50 (the CNN input); frames as in
 * noscope_diff_detect.  dds / cnns / result_host are host memory;
 * delta_cand, logit_cand, labels are device.  Synchronous.  Returns
 * NOSCOPE_INFEASIBLE (result = best-effort) when no pair meets the limits.   */
typedef struct {
  const noscope_dd_config* dd;   /* host pointer to the DD configuration      */
  const double* delta_cand;      /* device, strictly ascending                */
  int32_t n_delta;
} noscope_cbo_dd;
typedef struct {
  const noscope_cnn_arch* arch;  /* host pointers                             */
  const noscope_cnn_weights* weights;
  uint64_t t_snn_ps;             /* measured per-frame cost of this CNN       */
} noscope_cbo_cnn;
typedef struct {
  int32_t dd, cnn;               /* chosen indices                            */
  noscope_sweep_best best;       /* that pair's sweep result                  */
} noscope_cbo_result;

size_t noscope_cbo_workspace_bytes(const noscope_cbo_cnn* cnns, int32_t n_cnn, int64_t n,
                                   int32_t n_delta_max, int32_t m);
noscope_status noscope_cbo_search(const noscope_cbo_dd* dds, int32_t n_dd, const noscope_cbo_cnn* cnns,
                                  int32_t n_cnn, const uint8_t* frames, noscope_frames_desc desc,
                                  int64_t n, const uint8_t* labels, const float* logit_cand, int32_t m,
                                  uint64_t t_mse_ps, uint64_t t_full_ps, uint64_t fp_limit,
                                  uint64_t fn_limit, noscope_cbo_result* result_host, void* ws,
                                  size_t ws_bytes, noscope_stream_t stream);

/* ---- Evaluation -----------------------------------
 * "comparing frames labeled by the reference model and NoScope in
 * 30 frame windows ... agree on the presence of the target object in 28 of the
 * 30 frames"; SPEC windowed_accuracy / fp_fn_rates S:523-540.  Consecutive
 * non-overlapping windows of `window` frames (final partial window dropped);
 * a window is correct iff >= agree_min frames agree (label != 0 on both sides
 * or on neither).  Confusion counts cover all n frames.  pred, ref: device u8
 * [n]; counts_host: host.  ws: >= 256 bytes of device scratch.  Synchronous. */
typedef struct {
  int64_t windows, correct_windows, tp, tn, fp, fn;
} noscope_eval_counts;
noscope_status noscope_eval_labels(const uint8_t* pred, const uint8_t* ref, int64_t n, int32_t window,
                                   int32_t agree_min, noscope_eval_counts* counts_host, void* ws,
                                   size_t ws_bytes, noscope_stream_t stream);

/* ---- Specialized-CNN training ----------------------
 * P:472-477 "RMSprop ... between one and five epochs ... early stopping";
 * P:855-860 cross-validation.  Reading R-25: fp32 forward/backward (input =
 * the inference normalisation, no bf16 rounding inside), loss = mean binary
 * cross-entropy of the logit against labels[i] != 0, RMSprop
 *   v <- rho v + (1-rho) g^2;  p <- p - lr g / (sqrt(v) + eps)
 * on every parameter, one step per mini-batch of `batch` frames (last partial).
 * Epoch e visits perms[e][0..n_train) (device int32 frame indices into small,
 * the shuffled order is the caller's).  An epoch's training loss is the mean
 * over its samples of the loss of their mini-batch before that batch's update;
 * after each epoch the mean loss over val_idx (cross-validation) is recorded.
 * Training stops after the first epoch e >= 1 whose training loss exceeds
 * epoch e-1's ("early stopping if the training loss increases",
 * S:317), or after cfg.epochs epochs; `params` is left holding the parameters
 * of the epoch with the lowest cross-validation loss (earliest on ties).
 * params: device fp32 [noscope_cnn_param_count] in this order, each row-major:
 *   for each conv layer l: w [Cout][3][3][Cin], b [Cout]; then fc1 w [D][K]
 *   ((h, w, c) feature order), fc1 b [D], fc2 w [D], fc2 b [1].
 * history_host: host double [2 * epochs] (train loss, val loss per epoch run);
 * epochs_run_host: host.  Convolutions and dense layers run as GEMMs on
 * explicit im2col rows on the tcgen05 tensor cores at fp32 accuracy (3xTF32);
 * everything else in this library's kernels.  Synchronous (one host sync per
 * epoch).                                                                    */
typedef struct {
  int32_t batch, epochs;   /* mini-batch size; maximum epochs (the paper's 1-5) */
  float lr, rho, eps;
} noscope_train_config;
int64_t noscope_cnn_param_count(const noscope_cnn_arch* arch);
size_t noscope_cnn_train_workspace_bytes(const noscope_cnn_arch* arch, int32_t batch);
noscope_status noscope_cnn_train(const noscope_cnn_arch* arch, const noscope_train_config* cfg, float* params,
                                 const uint8_t* small, int64_t small_pitch, const uint8_t* labels,
                                 const int32_t* perms, int64_t n_train, const int32_t* val_idx, int64_t n_val,
                                 double* history_host, int32_t* epochs_run_host, void* ws, size_t ws_bytes,
                                 noscope_stream_t stream);
/* Trained fp32 parameters -> the inference weight buffers of `weights_out`
 * (conv / FC weights rounded to bf16 RNE, biases fp32; the caller owns and
 * sizes the buffers as for noscope_specialized_infer).  Asynchronous.         */
noscope_status noscope_cnn_params_to_weights(const noscope_cnn_arch* arch, const float* params,
                                             const noscope_cnn_weights* weights_out, noscope_stream_t stream);

/* Test hooks (not part of the cascade contract).
 * noscope_debug_cnn_layout: internal CNN activation offsets (layer-level tests).
 * noscope_debug_tc_gemm: the training path's fp32-accurate tcgen05 GEMM
 * (3xTF32 split: x = tf32(x) + (x - tf32(x)), three tensor-core products
 * accumulated in fp32) on caller buffers: C[m*ldc + n] = sum_k A[m*sam + k*sak]
 * * B[n*sbn + k*sbk], all device fp32; part = split-K scratch of
 * noscope_debug_tc_gemm_part_floats(M, N, K) floats (nullable when 0).      */
int32_t noscope_debug_cnn_layout(const noscope_cnn_arch* arch, int64_t n_max, int64_t* out);
size_t noscope_debug_tc_gemm_part_floats(int32_t M, int32_t N, int64_t K);
int32_t noscope_debug_tc_gemm(const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn, int64_t sbk,
                              float* C, int64_t ldc, int32_t M, int32_t N, int64_t K, float* part,
                              noscope_stream_t stream);

/* Reads and clears the device status word in a workspace (synchronises). */
noscope_status noscope_check(void* ws, noscope_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* NOSCOPE_H_ */
