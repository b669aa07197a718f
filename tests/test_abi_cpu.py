"""CPU-side checks of the C-ABI boundary: the library builds, loads, and exports
every function include/noscope.h declares; host-side size queries and
validation work without a GPU (no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "noscope.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(noscope_[a-z_0-9]+)\s*\(", src)
    return sorted(set(n for n in names if n != "noscope_labeller_fn"))


@pytest.fixture(scope="module")
def lib():
    from paper_1703_02529_b200 import build
    build.build_all()
    from paper_1703_02529_b200 import noscope
    return noscope.lib()


def test_header_declares_the_four_entry_points():
    fns = _declared_functions()
    for f in ("noscope_diff_detect", "noscope_specialized_infer", "noscope_cascade_run",
              "noscope_threshold_sweep"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    for f in _declared_functions():
        assert hasattr(lib, f), f"{f} not exported"


def test_host_queries_without_gpu(lib):
    from paper_1703_02529_b200 import noscope as N
    assert lib.noscope_version() == 100
    assert lib.noscope_status_string(7) == b"no feasible threshold triple"
    dd = N.DD(mode=1, metric=1, grid=10, t_diff_frames=30, t_skip_frames=1)
    c = dd.c()
    # state = 30 ring frames of 7504 B + label history (K+1)*t_skip = 31
    assert lib.noscope_stream_state_bytes(ctypes.byref(c)) == (30 * 7504 + 31 + 255) // 256 * 256
    arch = N.Arch(2, 32, 32).c()
    ws = lib.noscope_workspace_bytes(N.OP_CASCADE_RUN, ctypes.byref(c), ctypes.byref(arch), 108000, 0, 0)
    assert ws > 108000 * 7504
    assert lib.noscope_workspace_bytes(N.OP_SPECIALIZED_INFER, None, ctypes.byref(N.Arch(3, 32, 32).c()),
                                       10, 0, 0) == 0                  # unsupported arch
    assert lib.noscope_sweep_hist_words(100, 100) == 101 * 201 * 2 + 101 * 4 + 2
    bad = N.DD(mode=1, metric=1, grid=17).c()
    assert lib.noscope_stream_state_bytes(ctypes.byref(bad)) == 0      # grid > kMaxGrid


def test_validation_precedes_device_use(lib):
    from paper_1703_02529_b200 import noscope as N
    dd = N.DD(mode=0, metric=0, ref_image=None).c()                    # mode 0 needs ref image
    rc = lib.noscope_diff_detect(ctypes.byref(dd), None, N.FramesDesc(50, 50, 7504), 1, 0, None,
                                 None, 7504, None, None, None, None, None, 0, None)
    assert rc == 1
    dd = N.DD(mode=1, metric=0, out_w=60, out_h=60).c()
    rc = lib.noscope_diff_detect(ctypes.byref(dd), ctypes.c_void_p(16), N.FramesDesc(50, 50, 7504), 1,
                                 0, None, ctypes.c_void_p(16), 10816, None, ctypes.c_void_p(16),
                                 None, None, ctypes.c_void_p(16), 1 << 20, None)
    assert rc == 2                                                     # S:75 target > source
    dd = N.DD(mode=1, metric=0, out_w=53, out_h=720).c()                # u32 SSD would wrap
    rc = lib.noscope_diff_detect(ctypes.byref(dd), ctypes.c_void_p(16), N.FramesDesc(1280, 720, 2764800), 1,
                                 0, None, ctypes.c_void_p(16), 114480, None, ctypes.c_void_p(16),
                                 None, None, ctypes.c_void_p(16), 1 << 30, None)
    assert rc == 2
    dd = N.DD(mode=1, metric=0, out_w=50, out_h=50).c()                # 1920x1080: 126 KB band
    rc = lib.noscope_diff_detect(ctypes.byref(dd), ctypes.c_void_p(16), N.FramesDesc(1920, 1080, 6220800), 1,
                                 0, None, ctypes.c_void_p(16), 7504, None, ctypes.c_void_p(16),
                                 None, None, ctypes.c_void_p(16), 1 << 30, None)
    assert rc == 2
    rc = lib.noscope_threshold_sweep(4, None, None, None, None, 0, None, 1, None, 1, None, None, 0, 0,
                                     None, None, None, 0, None)
    assert rc == 1


def test_oracle_and_product_share_no_code():
    """The oracle never imports the CUDA path and vice versa (task rule ③)."""
    for d, forbidden in [("oracle", ("paper_1703_02529_b200",)),
                         ("paper_1703_02529_b200", ("oracle",))]:
        for dirpath, _, files in os.walk(os.path.join(ROOT, d)):
            for fn in files:
                if fn.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                    txt = open(os.path.join(dirpath, fn)).read()
                    for f in forbidden:
                        assert not re.search(rf"^\s*(from|import)\s+{f}\b", txt, re.M), (fn, f)
                        assert f"#include \"../../{f}" not in txt


def test_next_row_entry_points_validate_before_device_use(lib):
    """NEXT #1-#3 calls reject bad arguments on the host (no GPU needed)."""
    from paper_1703_02529_b200 import noscope as N
    v = ctypes.c_void_p(16)
    # fit workspace sizing: LR needs n*d doubles of z-scored features
    assert lib.noscope_fit_workspace_bytes(1000, 100, 7500) >= 1000 * 100 * 8
    assert lib.noscope_fit_workspace_bytes(-1, 100, 7500) == 0
    # reference image: null pointers / pitch not /16 / too-small workspace
    assert lib.noscope_reference_image(None, 7504, 50, 50, v, 10, v, v, 1 << 20, None) == 1
    assert lib.noscope_reference_image(v, 7501, 50, 50, v, 10, v, v, 1 << 20, None) == 2
    assert lib.noscope_reference_image(v, 7504, 50, 50, v, 10, v, v, 16, None) == 3
    # block features: grid above the 16x16 limit, mode 0 without a reference image
    dd = N.DD(mode=1, metric=1, grid=17, t_diff_frames=3).c()
    assert lib.noscope_block_features(ctypes.byref(dd), v, 7504, 4, v, None) == 2
    dd = N.DD(mode=0, metric=1, grid=10).c()
    assert lib.noscope_block_features(ctypes.byref(dd), v, 7504, 4, v, None) == 1
    # LR fit: n < 2 is a data error; l2 <= 0 (no minimiser), tol < 0 argument errors; d > 256 shape
    out = (ctypes.c_double * 3)()
    assert lib.noscope_lr_fit(v, v, 1, 2, 10, 1e-9, 0.1, out, None, v, 1 << 20, None) == 6
    assert lib.noscope_lr_fit(v, v, 10, 2, 10, 1e-9, -1.0, out, None, v, 1 << 20, None) == 1
    assert lib.noscope_lr_fit(v, v, 10, 2, 10, 1e-9, 0.0, out, None, v, 1 << 20, None) == 1
    assert lib.noscope_lr_fit(v, v, 10, 2, 10, -1.0, 0.1, out, None, v, 1 << 20, None) == 1
    assert lib.noscope_lr_fit(v, v, 10, 257, 10, 1e-9, 0.1, out, None, v, 1 << 20, None) == 2
    # eval: window / agree_min consistency
    cnt = N.EvalCounts()
    assert lib.noscope_eval_labels(v, v, 90, 30, 31, ctypes.byref(cnt), v, 256, None) == 1
    assert lib.noscope_eval_labels(v, v, 90, 0, 0, ctypes.byref(cnt), v, 256, None) == 1
    # CBO search: empty lists
    res = N.CboResult()
    assert lib.noscope_cbo_search(None, 0, None, 0, v, N.FramesDesc(50, 50, 7504), 10, v, v, 3, 1, 1, 0, 0,
                                  ctypes.byref(res), v, 1 << 20, None) == 1


def test_compact_fired_validates_before_device_use(lib):
    """noscope_compact_fired (H4 helper) rejects bad arguments on the host."""
    one = ctypes.c_void_p(16)
    ws = ctypes.c_void_p(256)
    big = 1 << 20
    assert lib.noscope_compact_fired(None, 10, 0, 1, one, one, ws, big, None) == 1        # null dispositions
    assert lib.noscope_compact_fired(one, 10, 0, 0, one, one, ws, big, None) == 1         # t_skip < 1
    assert lib.noscope_compact_fired(one, -1, 0, 1, one, one, ws, big, None) == 1         # n < 0
    assert lib.noscope_compact_fired(one, 1 << 31, 0, 1, one, one, ws, big, None) == 1    # n >= 2^31
    assert lib.noscope_compact_fired(one, 10, -1, 1, one, one, ws, big, None) == 1        # seg_offset < 0
    assert lib.noscope_compact_fired(one, 10, 0, 1, one, None, ws, big, None) == 1        # null count
    assert lib.noscope_compact_fired(one, 10, 0, 1, one, one, None, big, None) == 1       # null workspace
    need = lib.noscope_compact_workspace_bytes(1 << 20)
    assert lib.noscope_compact_fired(one, 1 << 20, 0, 1, one, one, ws, need - 1, None) == 3   # too small
    assert lib.noscope_compact_workspace_bytes(1 << 30) >= (1 << 30) // 8                # 1 bit per frame


def test_bench_reference_arm_prints_one_contract_line():
    """bench.py --impl reference (the CPU oracle arm the driver runs) prints one JSON
    line with the contract keys and an e2e object with zero copy bytes."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle"
