"""Thin Python binding of the C ABI in include/noscope.h (ctypes).

Argument marshalling only: every step of the hot path runs in libnoscope.so's
sm_100a kernels.  PyTorch supplies device memory (tensors) and the current CUDA
stream.  If the shared library is missing the import of the product path fails
loudly — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# NOSCOPE_LIB: an alternative build of the same sources (tools/ experiments)
LIB_PATH = os.environ.get("NOSCOPE_LIB") or os.path.join(_PKG, "libnoscope.so")

c_i32, c_i64, c_f32, c_f64, c_p, c_sz = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p, C.c_size_t

STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "SHAPE", 3: "WORKSPACE_TOO_SMALL", 4: "CUDA",
          5: "UNSUPPORTED_DEVICE", 6: "DATA", 7: "INFEASIBLE", 8: "LABELLER"}
OP_DIFF_DETECT, OP_SPECIALIZED_INFER, OP_CASCADE_RUN, OP_THRESHOLD_SWEEP = 0, 1, 2, 3
SKIPPED, SUPPRESSED, FIRED = 0, 1, 2
R_SKIP, R_SUPP, R_NEG, R_POS, R_UNC = 0, 1, 2, 3, 4


class NoScopeError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: {STATUS.get(code, code)} ({code})")
        self.code = code


class DDConfig(C.Structure):
    _fields_ = [("mode", c_i32), ("metric", c_i32), ("out_w", c_i32), ("out_h", c_i32),
                ("grid", c_i32), ("t_diff_frames", c_i32), ("t_skip_frames", c_i32),
                ("reserved", c_i32), ("delta_diff", c_f64), ("ref_image", c_p),
                ("lr_weights", c_p), ("lr_bias", c_f32), ("reserved2", c_f32)]


class FramesDesc(C.Structure):
    _fields_ = [("width", c_i32), ("height", c_i32), ("frame_pitch", c_i64)]


class CnnArchC(C.Structure):
    _fields_ = [("n_conv", c_i32), ("base_filters", c_i32), ("dense", c_i32), ("in_w", c_i32),
                ("in_h", c_i32), ("chan_mean", c_f32 * 3)]


class CnnWeightsC(C.Structure):
    _fields_ = [("conv_w", c_p * 4), ("conv_b", c_p * 4), ("fc1_w", c_p), ("fc1_b", c_p),
                ("fc2_w", c_p), ("fc2_b", c_p)]


class Route(C.Structure):
    _fields_ = [("lo_logit", c_f32), ("hi_logit", c_f32)]


class RunStats(C.Structure):
    _fields_ = [(n, c_i64) for n in ("n_frames", "n_skipped", "n_suppressed", "n_fired", "n_neg",
                                     "n_pos", "n_uncertain")]


class Timing(C.Structure):
    _fields_ = [("t_mse_ps", C.c_uint64), ("t_snn_ps", C.c_uint64), ("t_full_ps", C.c_uint64)]


class SweepBest(C.Structure):
    _fields_ = [("j", c_i32), ("l", c_i32), ("h", c_i32), ("feasible", c_i32),
                ("cost_ps", C.c_uint64), ("fp", C.c_uint64), ("fn", C.c_uint64),
                ("fired", C.c_uint64), ("uncertain", C.c_uint64), ("checked", C.c_uint64),
                ("total", C.c_uint64), ("delta", c_f64), ("lo_logit", c_f32), ("hi_logit", c_f32)]


class CboDD(C.Structure):
    _fields_ = [("dd", C.POINTER(DDConfig)), ("delta_cand", c_p), ("n_delta", c_i32)]


class CboCNN(C.Structure):
    _fields_ = [("arch", C.POINTER(CnnArchC)), ("weights", C.POINTER(CnnWeightsC)), ("t_snn_ps", C.c_uint64)]


class CboResult(C.Structure):
    _fields_ = [("dd", c_i32), ("cnn", c_i32), ("best", SweepBest)]


class EvalCounts(C.Structure):
    _fields_ = [(f, c_i64) for f in ("windows", "correct_windows", "tp", "tn", "fp", "fn")]


class TrainConfig(C.Structure):
    _fields_ = [("batch", c_i32), ("epochs", c_i32), ("lr", c_f32), ("rho", c_f32),
                ("eps", c_f32)]


class SweepTables(C.Structure):
    _fields_ = [(n, c_p) for n in ("F", "FPnf", "FNnf", "FPf", "FNf", "GE", "GT")]


LABELLER_FN = C.CFUNCTYPE(C.c_int, c_p, c_p, c_p, c_i64, c_i64, c_p, c_p)

_lib = None


def lib():
    """Load libnoscope.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1703_02529_b200.build`")
    L = C.CDLL(LIB_PATH)
    L.noscope_status_string.restype = C.c_char_p
    L.noscope_status_string.argtypes = [c_i32]
    L.noscope_version.restype = c_i32
    L.noscope_workspace_bytes.restype = c_sz
    L.noscope_workspace_bytes.argtypes = [c_i32, C.POINTER(DDConfig), C.POINTER(CnnArchC), c_i64,
                                          c_i32, c_i32]
    L.noscope_stream_state_bytes.restype = c_sz
    L.noscope_stream_state_bytes.argtypes = [C.POINTER(DDConfig)]
    L.noscope_stream_state_init.restype = c_i32
    L.noscope_stream_state_init.argtypes = [C.POINTER(DDConfig), c_p, c_p]
    L.noscope_sweep_hist_words.restype = c_sz
    L.noscope_sweep_hist_words.argtypes = [c_i32, c_i32]
    L.noscope_check.restype = c_i32
    L.noscope_check.argtypes = [c_p, c_p]
    L.noscope_diff_detect.restype = c_i32
    L.noscope_diff_detect.argtypes = [C.POINTER(DDConfig), c_p, FramesDesc, c_i64, c_i64, c_p, c_p,
                                      c_i64, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]
    L.noscope_specialized_infer.restype = c_i32
    L.noscope_specialized_infer.argtypes = [C.POINTER(CnnArchC), C.POINTER(CnnWeightsC), c_p, c_i64,
                                            c_p, c_p, c_i64, c_p, c_p, c_sz, c_p]
    L.noscope_route_logits.restype = c_i32
    L.noscope_route_logits.argtypes = [Route, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_sz, c_p]
    L.noscope_route_workspace_bytes.restype = c_sz
    L.noscope_route_workspace_bytes.argtypes = [c_i64]
    L.noscope_compact_fired.restype = c_i32
    L.noscope_compact_fired.argtypes = [c_p, c_i64, c_i64, c_i32, c_p, c_p, c_p, c_sz, c_p]
    L.noscope_compact_workspace_bytes.restype = c_sz
    L.noscope_compact_workspace_bytes.argtypes = [c_i64]
    L.noscope_cascade_run.restype = c_i32
    L.noscope_cascade_run.argtypes = [C.POINTER(DDConfig), C.POINTER(CnnArchC),
                                      C.POINTER(CnnWeightsC), Route, c_p, FramesDesc, c_i64, c_i64,
                                      c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p,
                                      C.POINTER(RunStats), c_p, c_sz, c_p]
    L.noscope_cascade_run_profiled.restype = c_i32
    L.noscope_cascade_run_profiled.argtypes = L.noscope_cascade_run.argtypes + [C.POINTER(c_f32)]
    L.noscope_launch_count.restype = C.c_uint64
    L.noscope_launch_count.argtypes = []
    L.noscope_threshold_sweep.restype = c_i32
    L.noscope_threshold_sweep.argtypes = [c_i32, c_p, c_p, c_p, c_p, c_i64, c_p, c_i32, c_p, c_i32,
                                          c_p, C.POINTER(Timing), C.c_uint64, C.c_uint64,
                                          C.POINTER(SweepTables), C.POINTER(SweepBest), c_p, c_sz,
                                          c_p]
    L.noscope_fit_workspace_bytes.restype = c_sz
    L.noscope_fit_workspace_bytes.argtypes = [c_i64, c_i32, c_i64]
    L.noscope_reference_image.restype = c_i32
    L.noscope_reference_image.argtypes = [c_p, c_i64, c_i32, c_i32, c_p, c_i64, c_p, c_p, c_sz, c_p]
    L.noscope_block_features.restype = c_i32
    L.noscope_block_features.argtypes = [C.POINTER(DDConfig), c_p, c_i64, c_i64, c_p, c_p]
    L.noscope_lr_fit.restype = c_i32
    L.noscope_lr_fit.argtypes = [c_p, c_p, c_i64, c_i32, c_i32, C.c_double, C.c_double,
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), c_p, c_sz, c_p]
    L.noscope_cbo_workspace_bytes.restype = c_sz
    L.noscope_cbo_workspace_bytes.argtypes = [C.POINTER(CboCNN), c_i32, c_i64, c_i32, c_i32]
    L.noscope_cbo_search.restype = c_i32
    L.noscope_cbo_search.argtypes = [C.POINTER(CboDD), c_i32, C.POINTER(CboCNN), c_i32, c_p, FramesDesc,
                                     c_i64, c_p, c_p, c_i32, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_uint64, C.POINTER(CboResult), c_p, c_sz, c_p]
    L.noscope_sweep_records.restype = c_i32
    L.noscope_sweep_records.argtypes = [c_p, c_p, c_i64, c_i32, c_i32, c_i32, c_p, c_p]
    L.noscope_eval_labels.restype = c_i32
    L.noscope_eval_labels.argtypes = [c_p, c_p, c_i64, c_i32, c_i32, C.POINTER(EvalCounts), c_p, c_sz, c_p]
    L.noscope_cnn_param_count.restype = c_i64
    L.noscope_cnn_param_count.argtypes = [C.POINTER(CnnArchC)]
    L.noscope_cnn_train_workspace_bytes.restype = c_sz
    L.noscope_cnn_train_workspace_bytes.argtypes = [C.POINTER(CnnArchC), c_i32]
    L.noscope_cnn_train.restype = c_i32
    L.noscope_cnn_train.argtypes = [C.POINTER(CnnArchC), C.POINTER(TrainConfig), c_p, c_p, c_i64, c_p, c_p, c_i64,
                                    c_p, c_i64, C.POINTER(C.c_double), C.POINTER(c_i32), c_p, c_sz, c_p]
    L.noscope_cnn_params_to_weights.restype = c_i32
    L.noscope_cnn_params_to_weights.argtypes = [C.POINTER(CnnArchC), c_p, C.POINTER(CnnWeightsC), c_p]
    L.noscope_debug_tc_gemm_part_floats.restype = c_sz
    L.noscope_debug_tc_gemm_part_floats.argtypes = [c_i32, c_i32, c_i64]
    L.noscope_debug_tc_gemm.restype = c_i32
    L.noscope_debug_tc_gemm.argtypes = [c_p, c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_i64, c_i32, c_i32, c_i64, c_p,
                                        c_p]
    L.noscope_debug_cnn_layout.restype = c_i32
    L.noscope_debug_cnn_layout.argtypes = [C.POINTER(CnnArchC), c_i64, C.POINTER(c_i64)]
    _lib = L
    return L


EXPORTED = ["noscope_status_string", "noscope_version", "noscope_workspace_bytes",
            "noscope_stream_state_bytes", "noscope_stream_state_init", "noscope_sweep_hist_words",
            "noscope_diff_detect", "noscope_specialized_infer", "noscope_route_logits",
            "noscope_cascade_run", "noscope_threshold_sweep", "noscope_check"]


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _check(code, where):
    if code != 0:
        raise NoScopeError(code, where)


# ------------------------------------------------------------------ configs
@dataclasses.dataclass
class DD:
    """Difference-detector configuration (mirrors noscope_dd_config)."""
    mode: int = 0
    metric: int = 0
    out_w: int = 50
    out_h: int = 50
    grid: int = 1
    t_diff_frames: int = 1
    t_skip_frames: int = 1
    delta_diff: float = 0.0
    ref_image: torch.Tensor | None = None      # cuda uint8 [out_h, out_w, 3]
    lr_weights: torch.Tensor | None = None     # cuda float32 [grid*grid]
    lr_bias: float = 0.0

    def c(self):
        return DDConfig(self.mode, self.metric, self.out_w, self.out_h, self.grid,
                        self.t_diff_frames, self.t_skip_frames, 0, float(self.delta_diff),
                        None if self.ref_image is None else self.ref_image.data_ptr(),
                        None if self.lr_weights is None else self.lr_weights.data_ptr(),
                        float(self.lr_bias), 0.0)


@dataclasses.dataclass
class Arch:
    n_conv: int
    base_filters: int
    dense: int
    in_w: int = 50
    in_h: int = 50
    chan_mean: tuple = (127.5, 127.5, 127.5)

    def c(self):
        return CnnArchC(self.n_conv, self.base_filters, self.dense, self.in_w, self.in_h,
                        (c_f32 * 3)(*self.chan_mean))


class Weights:
    """Device copies of a weight dict in the ABI layout (see synthgen.weights)."""

    def __init__(self, w: dict, device="cuda"):
        self.conv_w = [torch.from_numpy(a.view("int16")).to(device) for a in w["conv_w"]]
        self.conv_b = [torch.from_numpy(a).to(device) for a in w["conv_b"]]
        self.fc1_w = torch.from_numpy(w["fc1_w"].view("int16")).to(device)
        self.fc1_b = torch.from_numpy(w["fc1_b"]).to(device)
        self.fc2_w = torch.from_numpy(w["fc2_w"].view("int16")).to(device)
        self.fc2_b = torch.from_numpy(w["fc2_b"]).to(device)

    def c(self):
        cw = (c_p * 4)(*([t.data_ptr() for t in self.conv_w] + [None] * (4 - len(self.conv_w))))
        cb = (c_p * 4)(*([t.data_ptr() for t in self.conv_b] + [None] * (4 - len(self.conv_b))))
        return CnnWeightsC(cw, cb, self.fc1_w.data_ptr(), self.fc1_b.data_ptr(),
                           self.fc2_w.data_ptr(), self.fc2_b.data_ptr())


def small_pitch(out_w=50, out_h=50):
    return (out_w * out_h * 3 + 15) // 16 * 16


def workspace(op, dd=None, arch=None, n=0, n_delta=0, m=0, device="cuda"):
    b = lib().noscope_workspace_bytes(op, None if dd is None else C.byref(dd.c()),
                                      None if arch is None else C.byref(arch.c()), n, n_delta, m)
    if b == 0:
        raise NoScopeError(1, "noscope_workspace_bytes")
    return torch.empty(b, dtype=torch.uint8, device=device)


def noscope_stream_state_init(dd: DD, device="cuda", stream=None):
    c = dd.c()
    nb = lib().noscope_stream_state_bytes(C.byref(c))
    state = torch.empty(max(nb, 16), dtype=torch.uint8, device=device)
    _check(lib().noscope_stream_state_init(C.byref(c), _ptr(state), _stream(stream)),
           "noscope_stream_state_init")
    return state


# ------------------------------------------------------------------ entry points
def noscope_diff_detect(dd: DD, frames: torch.Tensor, width: int, height: int, seg_offset=0,
                        state=None, ws=None, small_out=None, stream=None, compact=True):
    """frames: cuda uint8 [n, frame_pitch].  Returns dict(small, score, disp, idx, n_fired)."""
    n, pitch = frames.shape
    dev = frames.device
    sp = small_pitch(dd.out_w, dd.out_h)
    small = small_out if small_out is not None else torch.empty((n, sp), dtype=torch.uint8, device=dev)
    score = torch.empty(n, dtype=torch.float64, device=dev)
    disp = torch.empty(n, dtype=torch.uint8, device=dev)
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=dev) if compact else None
    cnt = torch.zeros(1, dtype=torch.int64, device=dev) if compact else None
    if ws is None:
        ws = workspace(OP_DIFF_DETECT, dd, None, n, device=dev)
    _check(lib().noscope_diff_detect(C.byref(dd.c()), _ptr(frames), FramesDesc(width, height, pitch),
                                     n, seg_offset, _ptr(state), _ptr(small), sp, _ptr(score),
                                     _ptr(disp), _ptr(idx), _ptr(cnt), _ptr(ws), ws.numel(),
                                     _stream(stream)), "noscope_diff_detect")
    return dict(small=small, score=score, disp=disp, idx=idx, n_fired=cnt)


def noscope_specialized_infer(arch: Arch, weights: Weights, small: torch.Tensor, idx=None,
                              n_dev=None, n_max=None, ws=None, logits=None, stream=None):
    """small: cuda uint8 [*, small_pitch] (50x50x3 frames).  Returns fp32 logits [n_max]."""
    n_max = (idx.numel() if idx is not None else small.shape[0]) if n_max is None else n_max
    dev = small.device
    out = logits if logits is not None else torch.empty(max(n_max, 1), dtype=torch.float32, device=dev)
    if ws is None:
        ws = workspace(OP_SPECIALIZED_INFER, None, arch, n_max, device=dev)
    _check(lib().noscope_specialized_infer(C.byref(arch.c()), C.byref(weights.c()), _ptr(small),
                                           small.shape[1], _ptr(idx), _ptr(n_dev), n_max, _ptr(out),
                                           _ptr(ws), ws.numel(), _stream(stream)),
           "noscope_specialized_infer")
    return out[:n_max]


def noscope_route_logits(lo: float, hi: float, logits: torch.Tensor, n_dev=None, ws=None, out=None,
                         stream=None):
    """-> (route codes u8 [n], uncertain positions i32, count i64[1]); ws / out reusable."""
    n = logits.numel()
    dev = logits.device
    if ws is None:
        ws = torch.empty(lib().noscope_route_workspace_bytes(n), dtype=torch.uint8, device=dev)
    route, unc, nunc = out if out is not None else (
        torch.empty(max(n, 1), dtype=torch.uint8, device=dev), torch.empty(max(n, 1), dtype=torch.int32, device=dev),
        torch.zeros(1, dtype=torch.int64, device=dev))
    _check(lib().noscope_route_logits(Route(lo, hi), _ptr(logits), _ptr(n_dev), n, _ptr(route),
                                      _ptr(unc), _ptr(nunc), _ptr(ws), ws.numel(), _stream(stream)),
           "noscope_route_logits")
    return route[:n], unc, nunc


def noscope_compact_fired(disposition: torch.Tensor, seg_offset=0, t_skip=1, ws=None, out=None, stream=None):
    """Stable list of FIRED positions (disposition u8, rewritten in place for t_skip).
    -> (indices i32, count i64[1]); ws / out reusable."""
    n = disposition.numel()
    dev = disposition.device
    if ws is None:
        ws = torch.empty(lib().noscope_compact_workspace_bytes(n), dtype=torch.uint8, device=dev)
    idx, cnt = out if out is not None else (torch.empty(max(n, 1), dtype=torch.int32, device=dev),
                                            torch.zeros(1, dtype=torch.int64, device=dev))
    _check(lib().noscope_compact_fired(_ptr(disposition), n, seg_offset, t_skip, _ptr(idx), _ptr(cnt),
                                       _ptr(ws), ws.numel(), _stream(stream)), "noscope_compact_fired")
    return idx, cnt


def noscope_cascade_run(dd: DD, arch: Arch, weights: Weights, lo: float, hi: float,
                        frames: torch.Tensor, width: int, height: int, state: torch.Tensor,
                        labeller, labeller_user, seg_offset=0, frame_index_base=0, ws=None,
                        labels=None, route_out=None, logits_out=None, scores_out=None,
                        want_stats=False, stream=None, stage_ms=None):
    """One chunk of one unit through the whole cascade.

    labeller: an int function address (e.g. the stand-in from synthgen) or a
    LABELLER_FN instance; labeller_user: its void* (e.g. a device tensor).
    stage_ms: optional list; if given, the profiled entry point fills it with
    the 7 per-stage device times (ms) of noscope_cascade_run_profiled."""
    n, pitch = frames.shape
    dev = frames.device
    if ws is None:
        ws = workspace(OP_CASCADE_RUN, dd, arch, n, device=dev)
    labels = labels if labels is not None else torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    stats = RunStats() if want_stats else None
    fn = labeller if isinstance(labeller, int) else C.cast(labeller, c_p).value
    user = labeller_user.data_ptr() if isinstance(labeller_user, torch.Tensor) else labeller_user
    args = [C.byref(dd.c()), C.byref(arch.c()), C.byref(weights.c()), Route(lo, hi), _ptr(frames),
            FramesDesc(width, height, pitch), n, seg_offset, frame_index_base, _ptr(state),
            C.c_void_p(fn), C.c_void_p(user), _ptr(labels), _ptr(route_out), _ptr(logits_out),
            _ptr(scores_out), C.byref(stats) if stats is not None else None, _ptr(ws), ws.numel(),
            _stream(stream)]
    if stage_ms is None:
        code = lib().noscope_cascade_run(*args)
    else:
        buf = (c_f32 * 7)()
        code = lib().noscope_cascade_run_profiled(*args, buf)
        stage_ms[:] = list(buf)
    _check(code, "noscope_cascade_run")
    out = dict(labels=labels[:n], route=route_out, logits=logits_out, scores=scores_out)
    if stats is not None:
        out["stats"] = {f: getattr(stats, f) for f, _ in RunStats._fields_}
    return out


def launch_count():
    return int(lib().noscope_launch_count())


def sweep_hist_words(n_delta, m):
    return lib().noscope_sweep_hist_words(n_delta, m)


def noscope_threshold_sweep(phase, s, z, y, a, delta, u, hist, timing=(0, 0, 0), fp_limit=0,
                            fn_limit=0, tables=None, ws=None, stream=None, best_out=None):
    """phase 1: accumulate records into hist (uint64 tensor; viewed as int64 here);
    phase 2: evaluate hist -> (best dict, status); phase 3 both.
    best_out: a SweepBest in page-locked memory (pinned_sweep_best()) -> phase 2 is
    asynchronous (NOSCOPE_SWEEP_ASYNC); returns (best_out, 0) and best_out is valid
    after the stream synchronises (sweep_best_dict(best_out))."""
    nd, m = delta.numel(), u.numel()
    dev = delta.device
    if ws is None:
        ws = workspace(OP_THRESHOLD_SWEEP, None, None, 0, nd, m, device=dev)
    n = 0 if s is None else s.numel()
    best = best_out if best_out is not None else SweepBest()
    if best_out is not None and phase & 2:
        phase |= 4
    tab = None
    if tables is not None:
        tab = SweepTables(*[tables[k].data_ptr() for k in ("F", "FPnf", "FNnf", "FPf", "FNf", "GE", "GT")])
    tm = Timing(*[int(v) for v in timing])
    code = lib().noscope_threshold_sweep(phase, _ptr(s), _ptr(z), _ptr(y), _ptr(a), n, _ptr(delta),
                                         nd, _ptr(u), m, _ptr(hist), C.byref(tm), int(fp_limit),
                                         int(fn_limit), C.byref(tab) if tab is not None else None,
                                         C.byref(best) if phase & 2 else None, _ptr(ws), ws.numel(),
                                         _stream(stream))
    if code not in (0, 7):
        raise NoScopeError(code, "noscope_threshold_sweep")
    if not phase & 2:
        return None, code
    if best_out is not None:
        return best_out, code
    return sweep_best_dict(best), code


def sweep_best_dict(best):
    return {f: getattr(best, f) for f, _ in SweepBest._fields_}


def pinned_sweep_best():
    """A SweepBest living in page-locked host memory (target of an asynchronous phase 2)."""
    buf = torch.empty(C.sizeof(SweepBest), dtype=torch.uint8, pin_memory=True)
    best = SweepBest.from_address(buf.data_ptr())
    best._buf = buf    # keep the pinned storage alive
    return best


def noscope_sweep_records(s: torch.Tensor, y: torch.Tensor, mode: int, k: int, t_skip: int = 1, a_out=None,
                          stream=None):
    """a[i] = label emitted for record i when not fired (include/noscope.h)."""
    a_out = a_out if a_out is not None else torch.empty_like(y)
    _check(lib().noscope_sweep_records(_ptr(s), _ptr(y), s.numel(), mode, k, t_skip, _ptr(a_out),
                                       _stream(stream)), "noscope_sweep_records")
    return a_out


# ---------------------------------------------------------------- DD fitting
def fit_workspace(n, d, small_bytes, device="cuda"):
    nb = lib().noscope_fit_workspace_bytes(int(n), int(d), int(small_bytes))
    return torch.empty(max(nb, 256), dtype=torch.uint8, device=device)


def noscope_reference_image(small: torch.Tensor, labels: torch.Tensor, out_w=50, out_h=50, ref_out=None,
                            ws=None, stream=None):
    """small: device u8 [n, pitch]; labels: device u8 [n] -> device u8 [out_h*out_w*3]."""
    n, pitch = small.shape
    dev = small.device
    ref_out = ref_out if ref_out is not None else torch.empty(out_w * out_h * 3, dtype=torch.uint8, device=dev)
    ws = ws if ws is not None else fit_workspace(1, 1, out_w * out_h * 3, dev)
    _check(lib().noscope_reference_image(_ptr(small), pitch, out_w, out_h, _ptr(labels), n, _ptr(ref_out),
                                         _ptr(ws), ws.numel(), _stream(stream)), "noscope_reference_image")
    return ref_out


def noscope_block_features(dd: DD, small: torch.Tensor, n=None, feats=None, stream=None):
    """Per-frame block MSEs vs the anchor -> device f64 [n, grid*grid] (mode 1: rows < k NaN)."""
    n = small.shape[0] if n is None else n
    g = dd.grid
    feats = feats if feats is not None else torch.empty((n, g * g), dtype=torch.float64, device=small.device)
    _check(lib().noscope_block_features(C.byref(dd.c()), _ptr(small), small.shape[1], n, _ptr(feats),
                                        _stream(stream)), "noscope_block_features")
    return feats


def noscope_lr_fit(feats: torch.Tensor, targets: torch.Tensor, l2=None, tol=1e-9, max_iters=100, ws=None,
                   stream=None, info: dict | None = None):
    """feats: device f64 [n, d]; targets: device u8 [n] -> (w numpy f64 [d], b float), raw-feature
    form.  l2 defaults to 1/n (include/noscope.h).  `info` (optional dict) receives iters,
    grad_inf, J and stop."""
    n, d = feats.shape
    l2 = 1.0 / n if l2 is None else l2
    ws = ws if ws is not None else fit_workspace(n, d, 0, feats.device)
    out = (C.c_double * (d + 1))()
    inf = (C.c_double * 4)()
    _check(lib().noscope_lr_fit(_ptr(feats), _ptr(targets), n, d, int(max_iters), float(tol), float(l2), out,
                                inf, _ptr(ws), ws.numel(), _stream(stream)), "noscope_lr_fit")
    if info is not None:
        info.update(iters=int(inf[0]), grad_inf=inf[1], J=inf[2], stop=int(inf[3]))
    import numpy as np
    v = np.array(out[:], dtype=np.float64)
    return v[:d], float(v[d])


def noscope_cbo_search(dds, cnns, frames: torch.Tensor, width: int, height: int, labels: torch.Tensor,
                       logit_cand: torch.Tensor, t_mse_ps: int, t_full_ps: int, fp_limit: int, fn_limit: int,
                       stream=None):
    """dds: list of (DD, delta_cand device f64); cnns: list of (Arch, Weights, t_snn_ps).
    Returns (dd index, cnn index, best dict, status code 0 or 7)."""
    n, pitch = frames.shape
    keep = []                                  # keep the ctypes structs alive
    dd_arr = (CboDD * len(dds))()
    for i, (dd, dc) in enumerate(dds):
        c = dd.c()
        keep.append(c)
        dd_arr[i] = CboDD(C.pointer(c), dc.data_ptr(), dc.numel())
    cnn_arr = (CboCNN * len(cnns))()
    for i, (arch, w, t) in enumerate(cnns):
        ac, wc = arch.c(), w.c()
        keep += [ac, wc]
        cnn_arr[i] = CboCNN(C.pointer(ac), C.pointer(wc), int(t))
    ndm = max(dc.numel() for _, dc in dds)
    nb = lib().noscope_cbo_workspace_bytes(cnn_arr, len(cnns), n, ndm, logit_cand.numel())
    ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=frames.device)
    res = CboResult()
    code = lib().noscope_cbo_search(dd_arr, len(dds), cnn_arr, len(cnns), _ptr(frames),
                                    FramesDesc(width, height, pitch), n, _ptr(labels), _ptr(logit_cand),
                                    logit_cand.numel(), int(t_mse_ps), int(t_full_ps), int(fp_limit),
                                    int(fn_limit), C.byref(res), _ptr(ws), ws.numel(), _stream(stream))
    if code not in (0, 7):
        raise NoScopeError(code, "noscope_cbo_search")
    return res.dd, res.cnn, {f: getattr(res.best, f) for f, _ in SweepBest._fields_}, code


def noscope_eval_labels(pred: torch.Tensor, ref: torch.Tensor, window=30, agree_min=28, stream=None):
    """Windowed accuracy + confusion counts of device u8 label tracks -> dict."""
    ws = torch.empty(256, dtype=torch.uint8, device=pred.device)
    out = EvalCounts()
    _check(lib().noscope_eval_labels(_ptr(pred), _ptr(ref), pred.numel(), window, agree_min, C.byref(out),
                                     _ptr(ws), ws.numel(), _stream(stream)), "noscope_eval_labels")
    return {f: getattr(out, f) for f, _ in EvalCounts._fields_}


# ---------------------------------------------------------------- CNN training
def params_from_weight_dict(arch: Arch, w: dict, device="cuda"):
    """Host marshalling of a synthgen-layout weight dict (bf16 bits) into the
    flat fp32 parameter vector of noscope_cnn_train (header order)."""
    import numpy as np
    f32 = lambda bits: (np.asarray(bits, np.uint16).astype(np.uint32) << 16).view(np.float32).ravel()
    parts = []
    for l in range(arch.n_conv):
        parts += [f32(w["conv_w"][l]), np.asarray(w["conv_b"][l], np.float32).ravel()]
    parts += [f32(w["fc1_w"]), np.asarray(w["fc1_b"], np.float32).ravel(), f32(w["fc2_w"]),
              np.asarray(w["fc2_b"], np.float32).ravel()]
    v = np.concatenate(parts)
    assert v.size == lib().noscope_cnn_param_count(C.byref(arch.c()))
    return torch.from_numpy(v).to(device)


def noscope_cnn_train(arch: Arch, params: torch.Tensor, small: torch.Tensor, labels: torch.Tensor,
                      perms: torch.Tensor, val_idx: torch.Tensor, batch=32, lr=1e-3, rho=0.9, eps=1e-7,
                      stream=None):
    """params: device fp32 (updated in place to the best epoch's); perms: device int32
    [epochs, n_train]; val_idx: device int32 [n_val].  Returns (history, epochs_run)."""
    epochs, n_train = perms.shape
    ac = arch.c()
    nb = lib().noscope_cnn_train_workspace_bytes(C.byref(ac), batch)
    ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=params.device)
    cfg = TrainConfig(batch, epochs, lr, rho, eps)
    hist = (C.c_double * (2 * epochs))()
    run = c_i32(0)
    _check(lib().noscope_cnn_train(C.byref(ac), C.byref(cfg), _ptr(params), _ptr(small), small.shape[1],
                                   _ptr(labels), _ptr(perms), n_train, _ptr(val_idx), val_idx.numel(), hist,
                                   C.byref(run), _ptr(ws), ws.numel(), _stream(stream)), "noscope_cnn_train")
    return [(hist[2 * e], hist[2 * e + 1]) for e in range(run.value)], run.value


def noscope_cnn_params_to_weights(arch: Arch, params: torch.Tensor, weights: "Weights", stream=None):
    _check(lib().noscope_cnn_params_to_weights(C.byref(arch.c()), _ptr(params), C.byref(weights.c()),
                                               _stream(stream)), "noscope_cnn_params_to_weights")
    return weights


def noscope_check(ws, stream=None):
    return lib().noscope_check(_ptr(ws), _stream(stream))


def debug_tc_gemm(A: torch.Tensor, sam, sak, B: torch.Tensor, sbn, sbk, M, N, K, stream=None):
    """C [M, N] fp32 = sum_k A[m*sam + k*sak] * B[n*sbn + k*sbk] on the tcgen05 3xTF32 GEMM."""
    C = torch.empty((M, N), dtype=torch.float32, device=A.device)
    nf = lib().noscope_debug_tc_gemm_part_floats(M, N, K)
    part = torch.empty(max(nf, 1), dtype=torch.float32, device=A.device) if nf else None
    _check(lib().noscope_debug_tc_gemm(_ptr(A), sam, sak, _ptr(B), sbn, sbk, _ptr(C), N, M, N, K, _ptr(part),
                                       _stream(stream)), "noscope_debug_tc_gemm")
    return C


def debug_cnn_layout(arch: Arch, n_max: int):
    out = (c_i64 * 19)()
    _check(lib().noscope_debug_cnn_layout(C.byref(arch.c()), n_max, out), "debug_cnn_layout")
    return list(out)
