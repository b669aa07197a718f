"""GPU side of the synthetic input generator (harness, not the method).

Renders the same frames as synthgen.render_frames directly into HBM (the
decode stand-in, untimed) and exposes the ground-truth stand-in labeller as a
C function pointer compatible with noscope_labeller_fn."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import Scene

_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_DIR, "libsynthgen.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1703_02529_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.synth_render_bg.restype = C.c_int
        L.synth_render_bg.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]
        L.synth_render.restype = C.c_int
        L.synth_render.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                   C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def truth_labeller_address() -> int:
    """Address of synth_truth_labeller (user pointer = device uint8 truth track)."""
    return C.cast(lib().synth_truth_labeller, C.c_void_p).value


class GpuScene:
    """Device-resident event table / active slots / background for one stream."""

    def __init__(self, scene: Scene, device="cuda"):
        self.scene = scene
        sp = scene.spec
        self.events = torch.from_numpy(np.ascontiguousarray(scene.events).reshape(-1)).to(device)
        if self.events.numel() == 0:
            self.events = torch.zeros(10, dtype=torch.int32, device=device)
        self.active = torch.from_numpy(np.ascontiguousarray(scene.active)).to(device)
        self.truth = torch.from_numpy(scene.truth).to(device)
        self.bg = torch.empty(sp.height * sp.width * 3, dtype=torch.uint8, device=device)
        s = torch.cuda.current_stream().cuda_stream
        assert lib().synth_render_bg(self.bg.data_ptr(), sp.width, sp.height, sp.seed, sp.stream,
                                     C.c_void_p(s)) == 0

    def render(self, out: torch.Tensor, t_begin: int, n: int, stream=None):
        """Render frames t_begin..t_begin+n-1 into out (uint8 [>=n, pitch])."""
        sp = self.scene.spec
        s = (torch.cuda.current_stream() if stream is None else stream).cuda_stream
        assert out.shape[0] >= n and out.dtype == torch.uint8
        rc = lib().synth_render(out.data_ptr(), out.shape[1], sp.width, sp.height, t_begin, n,
                                sp.seed, sp.stream, sp.noise_sigma, self.bg.data_ptr(),
                                self.events.data_ptr(), self.active.data_ptr(), C.c_void_p(s))
        assert rc == 0
        return out
