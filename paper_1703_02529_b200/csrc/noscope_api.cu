// noscope_api.cu — the C ABI (include/noscope.h): host-side validation,
// workspace carving and launch sequencing.  No torch types cross this boundary.
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace ns {
bool cnn_arch_supported(const noscope_cnn_arch& a);
bool cnn_debug_layout(const noscope_cnn_arch& a, int64_t n_max, int64_t* out);
}  // namespace ns

using namespace ns;

namespace {

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

noscope_status check_device() {
  static DeviceInt cached;   // 1 supported, 2 not, per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return NOSCOPE_CUDA;
  int c = cached.get();
  if (c == 0) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return NOSCOPE_CUDA;
    c = (p.major == 10 && p.minor == 0) ? 1 : 2;
    cached.set(c);
  }
  return c == 1 ? NOSCOPE_OK : NOSCOPE_UNSUPPORTED_DEVICE;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

noscope_status validate_dd(const noscope_dd_config* c, bool check_ptrs = true) {
  if (!c) return NOSCOPE_INVALID_ARGUMENT;
  if (c->mode != 0 && c->mode != 1) return NOSCOPE_INVALID_ARGUMENT;
  if (c->metric != 0 && c->metric != 1) return NOSCOPE_INVALID_ARGUMENT;
  if (c->out_w < 1 || c->out_h < 1 || c->out_w > kMaxOutW) return NOSCOPE_SHAPE;
  // per-frame / per-block SSDs are u32: out_w*out_h*3 values of at most 255^2
  if ((int64_t)c->out_w * c->out_h * 3 * 65025 >= ((int64_t)1 << 32)) return NOSCOPE_SHAPE;
  if (c->t_skip_frames < 1) return NOSCOPE_INVALID_ARGUMENT;
  if (c->mode == 1 && c->t_diff_frames < 1) return NOSCOPE_INVALID_ARGUMENT;
  if (check_ptrs && c->mode == 0 && !c->ref_image) return NOSCOPE_INVALID_ARGUMENT;
  if (c->metric == 1) {
    if (c->grid < 1 || c->grid > kMaxGrid || c->grid > c->out_w || c->grid > c->out_h)
      return NOSCOPE_SHAPE;
    if (check_ptrs && !c->lr_weights) return NOSCOPE_INVALID_ARGUMENT;
  }
  if (std::isnan(c->delta_diff)) return NOSCOPE_INVALID_ARGUMENT;
  return NOSCOPE_OK;
}

noscope_status validate_frames(const noscope_dd_config* c, const noscope_frames_desc& d) {
  if (d.width < 1 || d.height < 1) return NOSCOPE_SHAPE;
  if (c->out_w > d.width || c->out_h > d.height) return NOSCOPE_SHAPE;
  if (d.frame_pitch % 16 != 0 || d.frame_pitch < (((int64_t)d.width * d.height * 3 + 15) & ~15ll))
    return NOSCOPE_SHAPE;
  // vertical box height must fit the 16-bit SWAR lanes (<= 257 rows of 255)
  const int64_t box_h = (d.height + c->out_h - 1) / c->out_h;
  const int64_t box_w = (d.width + c->out_w - 1) / c->out_w;
  if (box_h > 257 || box_h * box_w > kMaxBox) return NOSCOPE_SHAPE;
  // one band (box_h source rows) per ring stage, >= 2 stages per worker group:
  // bands up to ~110 KB (every source in PAPER.md Table 1, up to 1170x1080 -> 50x50)
  if (!dd_frames_fit(*c, d)) return NOSCOPE_SHAPE;
  return NOSCOPE_OK;
}

noscope_status validate_arch(const noscope_cnn_arch* a, const noscope_cnn_weights* w) {
  if (!a || !w) return NOSCOPE_INVALID_ARGUMENT;
  if (!cnn_arch_supported(*a)) return NOSCOPE_SHAPE;
  for (int l = 0; l < a->n_conv; ++l)
    if (!w->conv_w[l] || !w->conv_b[l]) return NOSCOPE_INVALID_ARGUMENT;
  if (!w->fc1_w || !w->fc1_b || !w->fc2_w || !w->fc2_b) return NOSCOPE_INVALID_ARGUMENT;
  return NOSCOPE_OK;
}

// ---- workspace layouts
struct DDWs {
  size_t status, scan, score, flags, total;
};
DDWs dd_ws(int64_t n) {
  DDWs w{};
  w.status = 0;
  w.scan = 256;
  w.score = w.scan + align256(compact_ws_bytes(n));
  w.flags = w.score + align256((size_t)n * 8);
  w.total = w.flags + align256(dd_flags_bytes());
  return w;
}

// Overlapped cascade (cascade_front_overlapped; opt-in, NOSCOPE_OVERLAP=1): for calls
// of at least kOverlapMinFrames frames whose CNN has a queue mode, the conv1+conv2
// kernel runs on kSideSms SMs beside dd_kernel (which leaves them free), consuming
// the fired frames as dd_kernel publishes them; what is left when the DD ends runs
// on the whole GPU.  Results are identical to the serial schedule; it is not the
// default because on B200 it is not faster: with the side SMs computing, dd_kernel
// (power-capped, HBM-bound) slows by as much as the CNN time it hides.
constexpr int64_t kOverlapMinFrames = 8192;
constexpr int kSideSms = 8;
bool overlap_requested() {
  const char* e = std::getenv("NOSCOPE_OVERLAP");
  return e && e[0] == '1';
}
bool overlap_sized(const noscope_cnn_arch* a, int64_t n) {
  return a && n >= kOverlapMinFrames && cnn_queue_supported(*a) && overlap_requested();
}

struct CascadeWs {
  size_t status, scan, small, score, disp, idx, nfired, logits, route_pf, unc, nunc, unc_pos,
      answers, counters, lab, flags, fq_head, fq, pos_pf, cnn, total;
  int64_t small_pitch;
};
// ovl: with the overlapped schedule's buffers (queue, per-frame positions, features of
// every queue slot)
CascadeWs cascade_ws(const noscope_dd_config* dd, const noscope_cnn_arch* a, int64_t n, bool ovl) {
  CascadeWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t r = off;
    off = align256(off + bytes);
    return r;
  };
  w.small_pitch = (small_bytes_of(*dd) + 15) & ~15ll;
  w.status = take(256);
  w.scan = take(compact_ws_bytes(n));
  w.small = take((size_t)n * w.small_pitch);
  w.score = take((size_t)n * 8);
  w.disp = take((size_t)n);
  w.idx = take((size_t)n * 4);
  w.nfired = take(8);
  w.logits = take((size_t)n * 4);
  w.route_pf = take((size_t)n);
  w.unc = take((size_t)n * 4);
  w.nunc = take(8);
  w.unc_pos = take((size_t)n * 4);
  w.answers = take((size_t)n);
  w.counters = take(64);
  w.lab = take(labels_ws_bytes(n));
  w.flags = take(dd_flags_bytes());
  w.fq_head = take(ovl ? kFqHeaderBytes : 0);
  w.fq = take(ovl ? (size_t)n * 4 : 0);
  w.pos_pf = take(ovl ? (size_t)n * 4 : 0);
  w.cnn = off;
  off += a ? std::max(cnn_ws_bytes(*a, n), ovl ? cnn_queue_ws_bytes(*a, n) : (size_t)0) : 0;
  w.total = align256(off);
  return w;
}

}  // namespace

extern "C" {

const char* noscope_status_string(noscope_status s) {
  switch (s) {
    case NOSCOPE_OK: return "ok";
    case NOSCOPE_INVALID_ARGUMENT: return "invalid argument";
    case NOSCOPE_SHAPE: return "shape error";
    case NOSCOPE_WORKSPACE_TOO_SMALL: return "workspace too small";
    case NOSCOPE_CUDA: return "CUDA error";
    case NOSCOPE_UNSUPPORTED_DEVICE: return "unsupported device (needs sm_100a / B200)";
    case NOSCOPE_DATA: return "NaN score or logit";
    case NOSCOPE_INFEASIBLE: return "no feasible threshold triple";
    case NOSCOPE_LABELLER: return "labeller callback failed";
  }
  return "unknown status";
}

int32_t noscope_version(void) { return 100; }

size_t noscope_stream_state_bytes(const noscope_dd_config* dd) {
  if (validate_dd(dd, false) != NOSCOPE_OK) return 0;
  return (size_t)align256(state_ring_bytes(*dd) + state_label_len(*dd));
}

noscope_status noscope_stream_state_init(const noscope_dd_config* dd, void* state,
                                         noscope_stream_t stream) {
  noscope_status s = validate_dd(dd, false);
  if (s != NOSCOPE_OK) return s;
  if (!state) return NOSCOPE_INVALID_ARGUMENT;
  if ((s = check_device()) != NOSCOPE_OK) return s;
  NS_CUDA_TRY(cudaMemsetAsync(state, 0, noscope_stream_state_bytes(dd), (cudaStream_t)stream));
  return NOSCOPE_OK;
}

size_t noscope_sweep_hist_words(int32_t nd, int32_t m) {
  if (nd < 1 || m < 1) return 0;
  return (size_t)(nd + 1) * (2 * m + 1) * 2 + (size_t)(nd + 1) * 4 + 2;
}

size_t noscope_workspace_bytes(noscope_op op, const noscope_dd_config* dd,
                               const noscope_cnn_arch* arch, int64_t n, int32_t nd, int32_t m) {
  if (n < 0) return 0;
  switch (op) {
    case NOSCOPE_OP_DIFF_DETECT:
      return dd_ws(n).total;
    case NOSCOPE_OP_SPECIALIZED_INFER:
      if (!arch || !cnn_arch_supported(*arch)) return 0;
      return 256 + cnn_ws_bytes(*arch, n);
    case NOSCOPE_OP_CASCADE_RUN:
      if (!arch || !dd || validate_dd(dd, false) != NOSCOPE_OK || !cnn_arch_supported(*arch))
        return 0;
      return cascade_ws(dd, arch, n, overlap_sized(arch, n)).total;
    case NOSCOPE_OP_THRESHOLD_SWEEP:
      if (nd < 1 || m < 1) return 0;
      return sweep_ws_bytes(nd, m);
  }
  return 0;
}

noscope_status noscope_check(void* ws, noscope_stream_t stream) {
  if (!ws) return NOSCOPE_INVALID_ARGUMENT;
  uint32_t st = 0;
  NS_CUDA_TRY(cudaMemcpyAsync(&st, ws, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  NS_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  NS_CUDA_TRY(cudaMemsetAsync(ws, 0, 4, (cudaStream_t)stream));
  return st ? NOSCOPE_DATA : NOSCOPE_OK;
}

noscope_status noscope_diff_detect(const noscope_dd_config* dd, const uint8_t* frames,
                                   noscope_frames_desc desc, int64_t n, int64_t seg_offset,
                                   void* state, uint8_t* small_out, int64_t small_pitch,
                                   double* score_out, uint8_t* disp_out, int32_t* fired_idx_out,
                                   int64_t* n_fired_dev, void* ws, size_t ws_bytes,
                                   noscope_stream_t stream) {
  noscope_status s = validate_dd(dd);
  if (s != NOSCOPE_OK) return s;
  if ((s = validate_frames(dd, desc)) != NOSCOPE_OK) return s;
  if (n < 0 || seg_offset < 0) return NOSCOPE_INVALID_ARGUMENT;
  if (!frames || !small_out || !disp_out || !ws) return NOSCOPE_INVALID_ARGUMENT;
  if ((fired_idx_out == nullptr) != (n_fired_dev == nullptr)) return NOSCOPE_INVALID_ARGUMENT;
  if (small_pitch % 16 || small_pitch < ((small_bytes_of(*dd) + 15) & ~15ll)) return NOSCOPE_SHAPE;
  if (!aligned16(frames) || !aligned16(small_out) || !aligned16(ws)) return NOSCOPE_INVALID_ARGUMENT;
  if (dd->mode == 1 && seg_offset > 0 && !state) return NOSCOPE_INVALID_ARGUMENT;
  DDWs w = dd_ws(n);
  if (ws_bytes < w.total) return NOSCOPE_WORKSPACE_TOO_SMALL;
  if ((s = check_device()) != NOSCOPE_OK) return s;
  if (n == 0) {
    if (n_fired_dev) NS_CUDA_TRY(cudaMemsetAsync(n_fired_dev, 0, 8, (cudaStream_t)stream));
    return NOSCOPE_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  uint32_t* status = reinterpret_cast<uint32_t*>(wsb + w.status);
  uint8_t* st8 = reinterpret_cast<uint8_t*>(state);
  if (!score_out) score_out = reinterpret_cast<double*>(wsb + w.score);
  s = launch_diff_detect(*dd, frames, desc, n, seg_offset, seg_offset > 0 ? st8 : nullptr, small_out,
                         small_pitch, score_out, disp_out, status,
                         reinterpret_cast<unsigned*>(wsb + w.flags), st);
  if (s != NOSCOPE_OK) return s;
  // compaction also fills skipped frames' disposition/score
  s = launch_compact_fired(disp_out, disp_out, score_out, n, seg_offset, dd->t_skip_frames,
                           fired_idx_out, n_fired_dev, wsb + w.scan, st);
  if (s != NOSCOPE_OK) return s;
  if (state && dd->mode == 1)
    s = launch_state_update(*dd, small_out, small_pitch, st8, seg_offset, n, nullptr, st);
  return s;
}

noscope_status noscope_specialized_infer(const noscope_cnn_arch* arch,
                                         const noscope_cnn_weights* weights,
                                         const uint8_t* small, int64_t small_pitch,
                                         const int32_t* idx, const int64_t* n_dev, int64_t n_max,
                                         float* logits, void* ws, size_t ws_bytes,
                                         noscope_stream_t stream) {
  noscope_status s = validate_arch(arch, weights);
  if (s != NOSCOPE_OK) return s;
  if (!small || !logits || !ws || n_max < 0) return NOSCOPE_INVALID_ARGUMENT;
  if (small_pitch % 16 || small_pitch < 7504) return NOSCOPE_SHAPE;
  if (!aligned16(small) || !aligned16(ws)) return NOSCOPE_INVALID_ARGUMENT;
  if (ws_bytes < noscope_workspace_bytes(NOSCOPE_OP_SPECIALIZED_INFER, nullptr, arch, n_max, 0, 0))
    return NOSCOPE_WORKSPACE_TOO_SMALL;
  if ((s = check_device()) != NOSCOPE_OK) return s;
  if (n_max == 0) return NOSCOPE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  const int64_t* nd = n_dev;
  if (!nd) {  // dense count: store n_max in the workspace header
    int64_t* hdr = reinterpret_cast<int64_t*>(wsb + 128);
    NS_CUDA_TRY(cudaMemcpyAsync(hdr, &n_max, 8, cudaMemcpyHostToDevice, st));
    nd = hdr;
  }
  return launch_cnn(*arch, *weights, small, small_pitch, idx, nd, n_max, logits, wsb + 256,
                    reinterpret_cast<uint32_t*>(wsb), st);
}

size_t noscope_route_workspace_bytes(int64_t n_max) { return compact_ws_bytes(std::max<int64_t>(n_max, 0)) + 256; }

noscope_status noscope_route_logits(noscope_route r, const float* logits, const int64_t* n_dev,
                                    int64_t n_max, uint8_t* route_out, int32_t* unc_idx_out,
                                    int64_t* n_unc_dev, void* ws, size_t ws_bytes, noscope_stream_t stream) {
  if (!(r.lo_logit <= r.hi_logit)) return NOSCOPE_INVALID_ARGUMENT;
  if ((!logits && n_max > 0) || !unc_idx_out || !n_unc_dev || n_max < 0 || !ws) return NOSCOPE_INVALID_ARGUMENT;
  if (!aligned16(ws)) return NOSCOPE_INVALID_ARGUMENT;
  if (ws_bytes < noscope_route_workspace_bytes(n_max)) return NOSCOPE_WORKSPACE_TOO_SMALL;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* b = reinterpret_cast<uint8_t*>(ws);
  uint32_t* status = reinterpret_cast<uint32_t*>(b);
  NS_CUDA_TRY(cudaMemsetAsync(status, 0, 4, st));
  return launch_route(r, logits, n_dev, n_max, nullptr, route_out, nullptr, unc_idx_out, n_unc_dev,
                      nullptr, nullptr, nullptr, b + 256, status, st);
}

size_t noscope_compact_workspace_bytes(int64_t n) { return compact_ws_bytes(std::max<int64_t>(n, 0)); }

noscope_status noscope_compact_fired(uint8_t* disposition, int64_t n, int64_t seg_offset,
                                     int32_t t_skip, int32_t* idx_out, int64_t* n_out_dev,
                                     void* ws, size_t ws_bytes, noscope_stream_t stream) {
  if (n < 0 || n >= ((int64_t)1 << 31) || t_skip < 1 || seg_offset < 0 || !n_out_dev || !ws)
    return NOSCOPE_INVALID_ARGUMENT;
  if (n > 0 && (!disposition || !idx_out)) return NOSCOPE_INVALID_ARGUMENT;
  if (!aligned16(ws)) return NOSCOPE_INVALID_ARGUMENT;
  if (ws_bytes < noscope_compact_workspace_bytes(n)) return NOSCOPE_WORKSPACE_TOO_SMALL;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  return launch_compact_fired(disposition, disposition, nullptr, n, seg_offset, t_skip, idx_out,
                              n_out_dev, ws, (cudaStream_t)stream);
}

// Overlap for this call?  Requested (NOSCOPE_OVERLAP=1), large, on the band-pipeline
// DD with a queue-mode CNN, outside stream capture (the side stream is created per
// call) and with a workspace sized for it (queried while the request was set).
static bool use_overlap(const noscope_dd_config* dd, const noscope_cnn_arch* arch,
                        const noscope_frames_desc& desc, int64_t n, cudaStream_t st) {
  if (!overlap_sized(arch, n) || !dd_uses_band_kernel(*dd, desc)) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
  return true;
}

static int side_sms() {
  int v = kSideSms;
  if (const char* e = std::getenv("NOSCOPE_SIDE_SMS")) v = std::max(0, std::min(32, std::atoi(e)));  // 0: no side kernel (A/B)
  return v;
}

// DD -> compaction -> CNN logits (compacted order) with the conv1+conv2 kernel
// overlapped with the DD:
//   main: fork | dd_kernel on (SMs - side) CTAs, appending fired frames to the queue
//   side:      | conv kernel, qmode 1, on `side` CTAs: claims published slots
//   main: conv kernel, qmode 2, whole GPU: the slots left when the DD ended
//         -> compaction (+ per-frame position) -> join side -> FC: slot p's logit to
//         logits[pos_pf[q[p]]], i.e. the same compacted order as the serial schedule.
static noscope_status cascade_front_overlapped(
    const noscope_dd_config* dd, const noscope_cnn_arch* arch, const noscope_cnn_weights* weights,
    const uint8_t* frames, const noscope_frames_desc& desc, int64_t n, int64_t seg_offset,
    uint8_t* st8, uint8_t* small, int64_t small_pitch, double* score, uint8_t* disp,
    uint32_t* status, int32_t* idx, int64_t* nfired, float* logits, uint8_t* b,
    const CascadeWs& w, cudaStream_t st, Prof* prof) {
  FiredQueue fq{};
  fq.q = reinterpret_cast<int32_t*>(b + w.fq);
  fq.count = reinterpret_cast<unsigned long long*>(b + w.fq_head);
  fq.claim = fq.count + 1;
  fq.done = reinterpret_cast<unsigned*>(fq.count + 2);
  int32_t* pos_pf = reinterpret_cast<int32_t*>(b + w.pos_pf);
  void* cws = b + w.cnn;
  NS_CUDA_TRY(cudaMemsetAsync(fq.count, 0, kFqHeaderBytes, st));
  NS_CUDA_TRY(cudaMemsetAsync(fq.q, 0xFF, (size_t)n * 4, st));   // -1: not yet published
  noscope_status s = cnn_queue_pack(*arch, *weights, n, cws, st);
  if (s != NOSCOPE_OK) return s;
  const int side = side_sms();
  cudaStream_t ss = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  auto cleanup = [&]() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (ss) cudaStreamDestroy(ss);   // released once its work completes
  };
  auto fail = [&](noscope_status e) {
    cleanup();
    return e;
  };
  if (cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(fork, st) != cudaSuccess)
    return fail(NOSCOPE_CUDA);
  s = launch_diff_detect(*dd, frames, desc, n, seg_offset, seg_offset > 0 ? st8 : nullptr, small,
                         small_pitch, score, disp, status, reinterpret_cast<unsigned*>(b + w.flags),
                         st, prof, &fq, side);  // e1
  if (s != NOSCOPE_OK) return fail(s);
  // the side kernel only after dd_kernel is enqueued (it waits for fq.producers CTAs)
  const bool side_on = fq.producers > 0 && side > 0;
  if (side_on) {
    if (cudaStreamWaitEvent(ss, fork, 0) != cudaSuccess) return fail(NOSCOPE_CUDA);
    s = cnn_queue_conv(*arch, *weights, small, small_pitch, fq, 1, side, n, cws, ss);
    if (s != NOSCOPE_OK) return fail(s);
    if (cudaEventRecord(join, ss) != cudaSuccess) return fail(NOSCOPE_CUDA);
  }
  int sms = kNumSMs;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device());
  s = cnn_queue_conv(*arch, *weights, small, small_pitch, fq, 2, sms, n, cws, st);
  if (s != NOSCOPE_OK) return fail(s);
  prof_mark(prof, st);  // e2
  s = launch_compact_fired(disp, disp, score, n, seg_offset, dd->t_skip_frames, idx, nfired,
                           b + w.scan, st, pos_pf);
  if (s != NOSCOPE_OK) return fail(s);
  prof_mark(prof, st);  // e3
  if (side_on && cudaStreamWaitEvent(st, join, 0) != cudaSuccess) return fail(NOSCOPE_CUDA);
  s = cnn_queue_fc(*arch, *weights, fq, n, pos_pf, logits, cws, st);
  if (s != NOSCOPE_OK) return fail(s);
  prof_mark(prof, st);  // e4
  cleanup();
  return NOSCOPE_OK;
}

static noscope_status cascade_impl(const noscope_dd_config* dd, const noscope_cnn_arch* arch,
                                   const noscope_cnn_weights* weights, noscope_route route,
                                   const uint8_t* frames, noscope_frames_desc desc, int64_t n,
                                   int64_t seg_offset, int64_t frame_index_base, void* state,
                                   noscope_labeller_fn labeller, void* labeller_user,
                                   uint8_t* labels_out, uint8_t* route_out, float* logits_out,
                                   double* scores_out, noscope_run_stats* stats_host, void* ws,
                                   size_t ws_bytes, noscope_stream_t stream, Prof* prof) {
  noscope_status s = validate_dd(dd);
  if (s != NOSCOPE_OK) return s;
  if ((s = validate_frames(dd, desc)) != NOSCOPE_OK) return s;
  if ((s = validate_arch(arch, weights)) != NOSCOPE_OK) return s;
  if (dd->out_w != arch->in_w || dd->out_h != arch->in_h) return NOSCOPE_SHAPE;
  if (!(route.lo_logit <= route.hi_logit)) return NOSCOPE_INVALID_ARGUMENT;
  if ((n > 0 && (!frames || !labels_out)) || !state || !labeller || !ws || n < 0 || seg_offset < 0)
    return NOSCOPE_INVALID_ARGUMENT;   // frames / labels may be null for an empty chunk
  if (!aligned16(frames) || !aligned16(ws) || !aligned16(state)) return NOSCOPE_INVALID_ARGUMENT;
  bool ovl = use_overlap(dd, arch, desc, n, (cudaStream_t)stream);
  CascadeWs w = cascade_ws(dd, arch, n, ovl);
  if (ovl && ws_bytes < w.total) {   // workspace sized for the serial schedule
    ovl = false;
    w = cascade_ws(dd, arch, n, false);
  }
  if (ws_bytes < w.total) return NOSCOPE_WORKSPACE_TOO_SMALL;
  if ((s = check_device()) != NOSCOPE_OK) return s;
  if (n == 0) {
    if (stats_host) std::memset(stats_host, 0, sizeof(*stats_host));
    return NOSCOPE_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* b = reinterpret_cast<uint8_t*>(ws);
  uint32_t* status = reinterpret_cast<uint32_t*>(b + w.status);
  uint8_t* small = b + w.small;
  double* score = scores_out ? scores_out : reinterpret_cast<double*>(b + w.score);
  uint8_t* disp = b + w.disp;
  int32_t* idx = reinterpret_cast<int32_t*>(b + w.idx);
  int64_t* nfired = reinterpret_cast<int64_t*>(b + w.nfired);
  float* logits = reinterpret_cast<float*>(b + w.logits);
  uint8_t* route_pf = b + w.route_pf;
  int32_t* unc = reinterpret_cast<int32_t*>(b + w.unc);
  int64_t* nunc = reinterpret_cast<int64_t*>(b + w.nunc);
  int32_t* unc_pos = reinterpret_cast<int32_t*>(b + w.unc_pos);
  uint8_t* answers = b + w.answers;
  uint64_t* counters = reinterpret_cast<uint64_t*>(b + w.counters);
  uint8_t* st8 = reinterpret_cast<uint8_t*>(state);

  NS_CUDA_TRY(cudaMemsetAsync(counters, 0, 64, st));
  prof_mark(prof, st);  // e0
  if (ovl) {
    s = cascade_front_overlapped(dd, arch, weights, frames, desc, n, seg_offset, st8, small,
                                 w.small_pitch, score, disp, status, idx, nfired, logits, b, w, st,
                                 prof);  // e1 .. e4
    if (s != NOSCOPE_OK) return s;
  } else {
  s = launch_diff_detect(*dd, frames, desc, n, seg_offset, seg_offset > 0 ? st8 : nullptr, small,
                         w.small_pitch, score, disp, status, reinterpret_cast<unsigned*>(b + w.flags),
                         st, prof);  // e1 after the fused downsample + score kernel
  if (s != NOSCOPE_OK) return s;
  prof_mark(prof, st);  // e2 (the separate lag-score stage no longer exists: ~0 ms)
  s = launch_compact_fired(disp, disp, score, n, seg_offset, dd->t_skip_frames, idx, nfired,
                           b + w.scan, st);
  if (s != NOSCOPE_OK) return s;
  prof_mark(prof, st);  // e3
  s = launch_cnn(*arch, *weights, small, w.small_pitch, idx, nfired, n, logits, b + w.cnn, status,
                 st);
  if (s != NOSCOPE_OK) return s;
  prof_mark(prof, st);  // e4
  }
  s = launch_route(route, logits, nfired, n, idx, nullptr, route_pf, unc, nunc, unc_pos, logits_out,
                   counters, b + w.scan, status, st);
  if (s != NOSCOPE_OK) return s;
  prof_mark(prof, st);  // e5
  if (labeller(labeller_user, unc, nunc, n, frame_index_base, answers, stream) != 0)
    return NOSCOPE_LABELLER;
  prof_mark(prof, st);  // e6
  const uint8_t* hist = seg_offset > 0 ? st8 + state_ring_bytes(*dd) : nullptr;
  s = launch_labels(*dd, seg_offset, n, disp, route_pf, unc_pos, answers, hist, labels_out,
                    route_out, b + w.lab, st);
  if (s != NOSCOPE_OK) return s;
  s = launch_state_update(*dd, small, w.small_pitch, st8, seg_offset, n, labels_out, st);
  if (s != NOSCOPE_OK) return s;
  prof_mark(prof, st);  // e7
  if (stats_host) {
    int64_t nf = 0, nu = 0;
    uint64_t cnt[2] = {0, 0};
    NS_CUDA_TRY(cudaMemcpyAsync(&nf, nfired, 8, cudaMemcpyDeviceToHost, st));
    NS_CUDA_TRY(cudaMemcpyAsync(&nu, nunc, 8, cudaMemcpyDeviceToHost, st));
    NS_CUDA_TRY(cudaMemcpyAsync(cnt, counters, 16, cudaMemcpyDeviceToHost, st));
    NS_CUDA_TRY(cudaStreamSynchronize(st));
    const int64_t ts = dd->t_skip_frames;
    const int64_t checked = (seg_offset + n + ts - 1) / ts - (seg_offset + ts - 1) / ts;
    stats_host->n_frames = n;
    stats_host->n_skipped = n - checked;
    stats_host->n_fired = nf;
    stats_host->n_suppressed = checked - nf;
    stats_host->n_neg = (int64_t)cnt[0];
    stats_host->n_pos = (int64_t)cnt[1];
    stats_host->n_uncertain = nu;
  }
  return NOSCOPE_OK;
}

noscope_status noscope_cascade_run(const noscope_dd_config* dd, const noscope_cnn_arch* arch,
                                   const noscope_cnn_weights* weights, noscope_route route,
                                   const uint8_t* frames, noscope_frames_desc desc, int64_t n,
                                   int64_t seg_offset, int64_t frame_index_base, void* state,
                                   noscope_labeller_fn labeller, void* labeller_user,
                                   uint8_t* labels_out, uint8_t* route_out, float* logits_out,
                                   double* scores_out, noscope_run_stats* stats_host, void* ws,
                                   size_t ws_bytes, noscope_stream_t stream) {
  return cascade_impl(dd, arch, weights, route, frames, desc, n, seg_offset, frame_index_base,
                      state, labeller, labeller_user, labels_out, route_out, logits_out,
                      scores_out, stats_host, ws, ws_bytes, stream, nullptr);
}

noscope_status noscope_cascade_run_profiled(
    const noscope_dd_config* dd, const noscope_cnn_arch* arch, const noscope_cnn_weights* weights,
    noscope_route route, const uint8_t* frames, noscope_frames_desc desc, int64_t n,
    int64_t seg_offset, int64_t frame_index_base, void* state, noscope_labeller_fn labeller,
    void* labeller_user, uint8_t* labels_out, uint8_t* route_out, float* logits_out,
    double* scores_out, noscope_run_stats* stats_host, void* ws, size_t ws_bytes,
    noscope_stream_t stream, float* stage_ms_host) {
  if (!stage_ms_host) return NOSCOPE_INVALID_ARGUMENT;
  Prof prof{};
  for (int i = 0; i < 8; ++i) NS_CUDA_TRY(cudaEventCreate(&prof.ev[i]));
  noscope_status s = cascade_impl(dd, arch, weights, route, frames, desc, n, seg_offset,
                                  frame_index_base, state, labeller, labeller_user, labels_out,
                                  route_out, logits_out, scores_out, stats_host, ws, ws_bytes,
                                  stream, &prof);
  if (s == NOSCOPE_OK && prof.n == 8) {
    NS_CUDA_TRY(cudaEventSynchronize(prof.ev[7]));
    for (int i = 0; i < 7; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prof.ev[i], prof.ev[i + 1]);
      stage_ms_host[i] = ms;
    }
  }
  for (int i = 0; i < 8; ++i) cudaEventDestroy(prof.ev[i]);
  return s;
}

uint64_t noscope_launch_count(void) { return ns::launch_counter(); }

noscope_status noscope_threshold_sweep(int32_t phase, const double* s, const float* z,
                                       const uint8_t* y, const uint8_t* a, int64_t n,
                                       const double* delta, int32_t nd, const float* u, int32_t m,
                                       uint64_t* hist, const noscope_timing* timing,
                                       uint64_t fp_limit, uint64_t fn_limit,
                                       const noscope_sweep_tables* tables,
                                       noscope_sweep_best* best_host, void* ws, size_t ws_bytes,
                                       noscope_stream_t stream) {
  const bool async_best = (phase & NOSCOPE_SWEEP_ASYNC) != 0;
  phase &= 3;
  if (phase < 1 || phase > 3) return NOSCOPE_INVALID_ARGUMENT;
  if (nd < 1 || m < 1 || m > 2048 || nd > 65535) return NOSCOPE_INVALID_ARGUMENT;
  if (!hist || !delta || !u || !ws) return NOSCOPE_INVALID_ARGUMENT;
  if ((phase & 1) && n > 0 && (!s || !z || !y || !a)) return NOSCOPE_INVALID_ARGUMENT;
  if ((phase & 2) && !timing) return NOSCOPE_INVALID_ARGUMENT;
  if (n < 0) return NOSCOPE_INVALID_ARGUMENT;
  if (ws_bytes < sweep_ws_bytes(nd, m)) return NOSCOPE_WORKSPACE_TOO_SMALL;
  noscope_status st = check_device();
  if (st != NOSCOPE_OK) return st;
  noscope_timing t0{0, 0, 0};
  bool infeasible = false;
  st = launch_sweep(phase, s, z, y, a, n, delta, nd, u, m, hist, timing ? *timing : t0, fp_limit,
                    fn_limit, tables, best_host, ws, (cudaStream_t)stream, async_best ? nullptr : &infeasible);
  if (st != NOSCOPE_OK) return st;
  return infeasible ? NOSCOPE_INFEASIBLE : NOSCOPE_OK;
}

// ---- DD fitting (fit.cu)
size_t noscope_fit_workspace_bytes(int64_t n, int32_t d, int64_t small_bytes) {
  if (n < 0 || d < 1 || small_bytes < 0) return 0;
  return fit_ws_bytes(n, d, small_bytes);
}

noscope_status noscope_reference_image(const uint8_t* small, int64_t small_pitch, int32_t out_w,
                                       int32_t out_h, const uint8_t* labels, int64_t n,
                                       uint8_t* ref_out, void* ws, size_t ws_bytes,
                                       noscope_stream_t stream) {
  if (!small || !labels || !ref_out || !ws || n < 0) return NOSCOPE_INVALID_ARGUMENT;
  if (out_w < 1 || out_h < 1) return NOSCOPE_SHAPE;
  const int64_t bytes = (int64_t)out_w * out_h * 3;
  if (small_pitch % 16 || small_pitch < ((bytes + 15) & ~15ll) || !aligned16(small)) return NOSCOPE_SHAPE;
  if (ws_bytes < fit_ws_bytes(1, 1, bytes)) return NOSCOPE_WORKSPACE_TOO_SMALL;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  if (n == 0) return NOSCOPE_DATA;
  uint64_t m = 0;
  s = launch_reference_image(small, small_pitch, (int)bytes, labels, n, ref_out, ws, &m,
                             (cudaStream_t)stream);
  if (s != NOSCOPE_OK) return s;
  return m == 0 ? NOSCOPE_DATA : NOSCOPE_OK;
}

noscope_status noscope_block_features(const noscope_dd_config* dd, const uint8_t* small,
                                      int64_t small_pitch, int64_t n, double* feats,
                                      noscope_stream_t stream) {
  if (!dd || !small || !feats || n < 0) return NOSCOPE_INVALID_ARGUMENT;
  if (dd->mode != 0 && dd->mode != 1) return NOSCOPE_INVALID_ARGUMENT;
  if (dd->mode == 0 && !dd->ref_image) return NOSCOPE_INVALID_ARGUMENT;
  if (dd->mode == 1 && dd->t_diff_frames < 1) return NOSCOPE_INVALID_ARGUMENT;
  if (dd->out_w < 1 || dd->out_h < 1) return NOSCOPE_SHAPE;
  if (dd->grid < 1 || dd->grid > kMaxGrid || dd->grid > dd->out_w || dd->grid > dd->out_h)
    return NOSCOPE_SHAPE;
  const int64_t bytes = (int64_t)dd->out_w * dd->out_h * 3;
  if (small_pitch % 16 || small_pitch < ((bytes + 15) & ~15ll)) return NOSCOPE_SHAPE;
  if (bytes * 65025 >= (int64_t)1 << 32) return NOSCOPE_SHAPE;   // u32 block SSD
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  if (n == 0) return NOSCOPE_OK;
  return launch_block_features(*dd, small, small_pitch, n, feats, (cudaStream_t)stream);
}

noscope_status noscope_lr_fit(const double* feats, const uint8_t* targets, int64_t n, int32_t d,
                              int32_t max_iters, double tol, double l2, double* w_host, double* info_host,
                              void* ws, size_t ws_bytes, noscope_stream_t stream) {
  if (!feats || !targets || !w_host || !ws || d < 1 || max_iters < 0 || !(tol >= 0) || !(l2 > 0) ||
      !std::isfinite(l2))
    return NOSCOPE_INVALID_ARGUMENT;
  if (d > 256) return NOSCOPE_SHAPE;
  if (n < 2) return NOSCOPE_DATA;
  if (ws_bytes < fit_ws_bytes(n, d, 0)) return NOSCOPE_WORKSPACE_TOO_SMALL;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  return launch_lr_fit(feats, targets, n, d, max_iters, tol, l2, w_host, info_host, ws, (cudaStream_t)stream);
}

// ---- Full CBO search (cbo.cu helper + the existing entry points)
namespace {
struct CboWs {
  size_t small, score, disp, a, logits, hist, dd, cnn, sweep, total;
  size_t cnn_bytes;
};
CboWs cbo_ws(const noscope_cbo_cnn* cnns, int32_t n_cnn, int64_t n, int32_t ndm, int32_t m) {
  CboWs w{};
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t r = off;
    off = align256(off + b);
    return r;
  };
  w.small = take((size_t)n * 7504);
  w.score = take((size_t)n * 8);
  w.disp = take((size_t)n);
  w.a = take((size_t)n);
  w.logits = take((size_t)n_cnn * n * 4);
  w.hist = take(noscope_sweep_hist_words(ndm, m) * 8);
  w.dd = take(dd_ws(n).total);
  size_t cb = 0;
  for (int c = 0; c < n_cnn; ++c)
    cb = std::max(cb, noscope_workspace_bytes(NOSCOPE_OP_SPECIALIZED_INFER, nullptr, cnns[c].arch, n, 0, 0));
  w.cnn_bytes = cb;
  w.cnn = take(cb);
  w.sweep = take(sweep_ws_bytes(ndm, m));
  w.total = off;
  return w;
}
}  // namespace

size_t noscope_cbo_workspace_bytes(const noscope_cbo_cnn* cnns, int32_t n_cnn, int64_t n,
                                   int32_t n_delta_max, int32_t m) {
  if (!cnns || n_cnn < 1 || n < 0 || n_delta_max < 1 || m < 1) return 0;
  for (int c = 0; c < n_cnn; ++c)
    if (!cnns[c].arch || !cnn_arch_supported(*cnns[c].arch)) return 0;
  return cbo_ws(cnns, n_cnn, n, n_delta_max, m).total;
}

noscope_status noscope_cbo_search(const noscope_cbo_dd* dds, int32_t n_dd, const noscope_cbo_cnn* cnns,
                                  int32_t n_cnn, const uint8_t* frames, noscope_frames_desc desc,
                                  int64_t n, const uint8_t* labels, const float* logit_cand, int32_t m,
                                  uint64_t t_mse_ps, uint64_t t_full_ps, uint64_t fp_limit,
                                  uint64_t fn_limit, noscope_cbo_result* result_host, void* ws,
                                  size_t ws_bytes, noscope_stream_t stream) {
  if (!dds || n_dd < 1 || !cnns || n_cnn < 1 || !frames || !labels || !logit_cand || m < 1 ||
      !result_host || !ws || n < 1)
    return NOSCOPE_INVALID_ARGUMENT;
  int32_t ndm = 0;
  for (int d = 0; d < n_dd; ++d) {
    if (!dds[d].dd || !dds[d].delta_cand || dds[d].n_delta < 1) return NOSCOPE_INVALID_ARGUMENT;
    if (dds[d].dd->out_w != 50 || dds[d].dd->out_h != 50) return NOSCOPE_SHAPE;
    noscope_status s = validate_dd(dds[d].dd);
    if (s != NOSCOPE_OK) return s;
    ndm = std::max(ndm, dds[d].n_delta);
  }
  const size_t need = noscope_cbo_workspace_bytes(cnns, n_cnn, n, ndm, m);
  if (need == 0) return NOSCOPE_SHAPE;
  if (ws_bytes < need) return NOSCOPE_WORKSPACE_TOO_SMALL;
  CboWs w = cbo_ws(cnns, n_cnn, n, ndm, m);
  uint8_t* b = reinterpret_cast<uint8_t*>(ws);
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* small = b + w.small;
  double* score = reinterpret_cast<double*>(b + w.score);
  uint8_t* a = b + w.a;
  uint64_t* hist = reinterpret_cast<uint64_t*>(b + w.hist);
  bool have = false;
  noscope_cbo_result best{};
  uint64_t bk[4] = {0, 0, 0, 0};
  // R-23: every CNN runs unfiltered on all n frames.  A DD launch writes only the
  // small frames its configuration needs (checked frames and their anchors), so
  // the CNN input comes from a t_skip = 1 pass of dds[0] (every frame checked,
  // every frame downsampled); the same 50x50 frames serve every DD config.
  auto cnn_pass = [&]() -> noscope_status {
    for (int c = 0; c < n_cnn; ++c) {
      noscope_status s = noscope_specialized_infer(cnns[c].arch, cnns[c].weights, small, 7504, nullptr, nullptr,
                                                   n, reinterpret_cast<float*>(b + w.logits) + (size_t)c * n,
                                                   b + w.cnn, w.cnn_bytes, stream);
      if (s != NOSCOPE_OK) return s;
    }
    return NOSCOPE_OK;
  };
  if (dds[0].dd->t_skip_frames != 1) {
    noscope_dd_config all = *dds[0].dd;
    all.t_skip_frames = 1;
    noscope_status s = noscope_diff_detect(&all, frames, desc, n, 0, nullptr, small, 7504, score, b + w.disp,
                                           nullptr, nullptr, b + w.dd, dd_ws(n).total, stream);
    if (s != NOSCOPE_OK) return s;
    if ((s = cnn_pass()) != NOSCOPE_OK) return s;
  }
  for (int d = 0; d < n_dd; ++d) {
    const noscope_dd_config& dd = *dds[d].dd;
    noscope_status s = noscope_diff_detect(&dd, frames, desc, n, 0, nullptr, small, 7504, score,
                                           b + w.disp, nullptr, nullptr, b + w.dd, dd_ws(n).total, stream);
    if (s != NOSCOPE_OK) return s;
    if (d == 0 && dd.t_skip_frames == 1 && (s = cnn_pass()) != NOSCOPE_OK) return s;
    s = launch_records_a(score, labels, n, dd.mode, dd.t_diff_frames, dd.t_skip_frames, a, st);
    if (s != NOSCOPE_OK) return s;
    for (int c = 0; c < n_cnn; ++c) {
      NS_CUDA_TRY(cudaMemsetAsync(hist, 0, noscope_sweep_hist_words(dds[d].n_delta, m) * 8, st));
      const noscope_timing tm{t_mse_ps, cnns[c].t_snn_ps, t_full_ps};
      noscope_sweep_best r{};
      s = noscope_threshold_sweep(3, score, reinterpret_cast<const float*>(b + w.logits) + (size_t)c * n,
                                  labels, a, n, dds[d].delta_cand, dds[d].n_delta, logit_cand, m, hist,
                                  &tm, fp_limit, fn_limit, nullptr, &r, b + w.sweep,
                                  sweep_ws_bytes(ndm, m), stream);
      if (s != NOSCOPE_OK && s != NOSCOPE_INFEASIBLE) return s;
      const uint64_t viol =
          r.feasible ? 0
                     : std::max<uint64_t>(r.fp > fp_limit ? r.fp - fp_limit : 0, r.fn > fn_limit ? r.fn - fn_limit : 0);
      const uint64_t key[4] = {r.feasible ? 0u : 1u, viol, r.cost_ps, r.uncertain};
      bool better = !have;
      for (int q = 0; q < 4 && !better; ++q) {
        if (key[q] < bk[q]) better = true;
        if (key[q] != bk[q]) break;
      }
      if (better) {   // ties keep the earlier (dd, cnn): iteration order is the key's tail
        have = true;
        std::memcpy(bk, key, sizeof(bk));
        best.dd = d;
        best.cnn = c;
        best.best = r;
      }
    }
  }
  *result_host = best;
  return best.best.feasible ? NOSCOPE_OK : NOSCOPE_INFEASIBLE;
}

noscope_status noscope_sweep_records(const double* s, const uint8_t* y, int64_t n, int32_t mode, int32_t k,
                                     int32_t t_skip, uint8_t* a_out, noscope_stream_t stream) {
  if ((n > 0 && (!s || !y || !a_out)) || n < 0 || (mode != 0 && mode != 1) || k < 1 || t_skip < 1)
    return NOSCOPE_INVALID_ARGUMENT;
  noscope_status st = check_device();
  if (st != NOSCOPE_OK) return st;
  return launch_records_a(s, y, n, mode, k, t_skip, a_out, (cudaStream_t)stream);
}

noscope_status noscope_eval_labels(const uint8_t* pred, const uint8_t* ref, int64_t n, int32_t window,
                                   int32_t agree_min, noscope_eval_counts* counts_host, void* ws,
                                   size_t ws_bytes, noscope_stream_t stream) {
  if (!pred || !ref || !counts_host || !ws || n < 0 || window < 1 || agree_min < 0 || agree_min > window)
    return NOSCOPE_INVALID_ARGUMENT;
  if (ws_bytes < 256) return NOSCOPE_WORKSPACE_TOO_SMALL;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  int64_t out[6];
  s = launch_eval_labels(pred, ref, n, window, agree_min, reinterpret_cast<unsigned long long*>(ws), out,
                         (cudaStream_t)stream);
  if (s != NOSCOPE_OK) return s;
  *counts_host = noscope_eval_counts{out[0], out[1], out[2], out[3], out[4], out[5]};
  return NOSCOPE_OK;
}

// ---- specialized-CNN training (train.cu)
int64_t noscope_cnn_param_count(const noscope_cnn_arch* arch) {
  if (!arch || !cnn_arch_supported(*arch)) return 0;
  return train_param_count(*arch);
}

size_t noscope_cnn_train_workspace_bytes(const noscope_cnn_arch* arch, int32_t batch) {
  if (!arch || !cnn_arch_supported(*arch) || batch < 1 || batch > 1024) return 0;
  return train_ws_bytes(*arch, batch);
}

noscope_status noscope_cnn_train(const noscope_cnn_arch* arch, const noscope_train_config* cfg, float* params,
                                 const uint8_t* small, int64_t small_pitch, const uint8_t* labels,
                                 const int32_t* perms, int64_t n_train, const int32_t* val_idx, int64_t n_val,
                                 double* history_host, int32_t* epochs_run_host, void* ws, size_t ws_bytes,
                                 noscope_stream_t stream) {
  if (!arch || !cfg || !params || !small || !labels || !perms || !history_host || !epochs_run_host || !ws)
    return NOSCOPE_INVALID_ARGUMENT;
  if (!cnn_arch_supported(*arch)) return NOSCOPE_SHAPE;
  if (cfg->batch < 1 || cfg->batch > 1024 || cfg->epochs < 1 || !(cfg->lr > 0) ||
      !(cfg->rho >= 0 && cfg->rho < 1) || !(cfg->eps > 0) || n_train < 1 || n_val < 0 || (n_val > 0 && !val_idx))
    return NOSCOPE_INVALID_ARGUMENT;
  if (small_pitch % 16 || small_pitch < 7504) return NOSCOPE_SHAPE;
  if (ws_bytes < train_ws_bytes(*arch, cfg->batch)) return NOSCOPE_WORKSPACE_TOO_SMALL;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  return launch_cnn_train(*arch, *cfg, params, small, small_pitch, labels, perms, n_train, val_idx, n_val,
                          history_host, epochs_run_host, ws, (cudaStream_t)stream);
}

noscope_status noscope_cnn_params_to_weights(const noscope_cnn_arch* arch, const float* params,
                                             const noscope_cnn_weights* weights_out, noscope_stream_t stream) {
  if (!arch || !params || !weights_out) return NOSCOPE_INVALID_ARGUMENT;
  if (!cnn_arch_supported(*arch)) return NOSCOPE_SHAPE;
  for (int l = 0; l < arch->n_conv; ++l)
    if (!weights_out->conv_w[l] || !weights_out->conv_b[l]) return NOSCOPE_INVALID_ARGUMENT;
  if (!weights_out->fc1_w || !weights_out->fc1_b || !weights_out->fc2_w || !weights_out->fc2_b)
    return NOSCOPE_INVALID_ARGUMENT;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  return launch_params_to_weights(*arch, params, *weights_out, (cudaStream_t)stream);
}

// Test/debug helper (not part of the four-call contract): internal CNN
// activation offsets within the specialized_infer workspace, so tests can
// check individual layers.  out[19]: per conv layer l = 0..3 {offset of its
// stacked input map (-1: not materialised), rows per plane, H, channels}, then
// feature-tile offset, K, chunk.  Offsets include the 256-B header.
int32_t noscope_debug_cnn_layout(const noscope_cnn_arch* arch, int64_t n_max, int64_t* out) {
  if (!arch || !out || !ns::cnn_debug_layout(*arch, n_max, out)) return 1;
  for (int i : {0, 4, 8, 12, 16})
    if (out[i] >= 0) out[i] += 256;
  return 0;
}

// Test/debug helper: the training path's fp32-accurate tcgen05 GEMM (gemm_tc.cu)
// on caller buffers, C[m*ldc + n] = sum_k A[m*sam + k*sak] * B[n*sbn + k*sbk]
// (device fp32); part: device scratch of noscope_debug_tc_gemm_part_floats(M, N,
// K) floats (nullable when 0).  Asynchronous.
size_t noscope_debug_tc_gemm_part_floats(int32_t M, int32_t N, int64_t K) {
  return ns::tc_gemm_part_floats(M, N, K);
}
int32_t noscope_debug_tc_gemm(const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbn, int64_t sbk,
                              float* C, int64_t ldc, int32_t M, int32_t N, int64_t K, float* part,
                              noscope_stream_t stream) {
  if (!A || !B || !C || M < 0 || N < 0 || K < 0) return NOSCOPE_INVALID_ARGUMENT;
  noscope_status s = check_device();
  if (s != NOSCOPE_OK) return s;
  return ns::tc_gemm(A, sam, sak, B, sbn, sbk, C, ldc, M, N, K, part, (cudaStream_t)stream);
}

}  // extern "C"
