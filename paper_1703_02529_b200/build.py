"""Build the in-tree shared libraries for sm_100a with nvcc.

  libnoscope.so   — the product: C ABI of include/noscope.h (csrc/*.cu)
  synthgen/libsynthgen.so — harness: GPU renderer of the synthetic video and
                    the ground-truth stand-in labeller (synthgen/synth_gpu.cu)

Both are built IN-TREE so they travel to the GPU box with the repo snapshot.
Usage: python -m paper_1703_02529_b200.build [--force]
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]

LIB_SOURCES = ["noscope_api.cu", "dd.cu", "scan.cu", "sweep.cu", "cnn.cu", "cnn_fused.cu", "cnn_gemm.cu", "cnn_tile.cu", "fit.cu", "cbo.cu", "train.cu", "gemm_tc.cu"]
LIB_HEADERS = ["common.cuh", "internal.h"]


def _digest(paths):
    h = hashlib.sha256()
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def _build(out, sources, deps, extra=()):
    stamp = out + ".sha"
    dig = _digest(list(sources) + list(deps))
    if os.path.exists(out) and os.path.exists(stamp) and open(stamp).read() == dig \
            and "--force" not in sys.argv:
        return out
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-o", out, *sources]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(dig)
    return out


def build_noscope():
    csrc = os.path.join(PKG, "csrc")
    srcs = [os.path.join(csrc, s) for s in LIB_SOURCES]
    deps = [os.path.join(csrc, h) for h in LIB_HEADERS] + [os.path.join(ROOT, "include", "noscope.h")]
    return _build(os.path.join(PKG, "libnoscope.so"), srcs, deps)


def build_synthgen():
    d = os.path.join(ROOT, "synthgen")
    src = os.path.join(d, "synth_gpu.cu")
    return _build(os.path.join(d, "libsynthgen.so"), [src], [])


def build_all():
    return build_noscope(), build_synthgen()


if __name__ == "__main__":
    for p in build_all():
        print(p)
