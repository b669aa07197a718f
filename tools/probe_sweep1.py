"""Host vs device time of a phase-1 threshold-sweep call on 1M records, with and
without a caller-provided workspace (diagnoses bench.py's sweep_1M hist_ms)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_1703_02529_b200 import noscope as N  # noqa: E402
rng = np.random.default_rng(4)
M = 1_000_000
y = (rng.random(M) < 0.15).astype(np.uint8)
s = np.where(rng.random(M) < 0.05, -np.inf, rng.gamma(2.0, 10.0, M) + 40.0 * y)
z = (rng.normal(0, 1, M) + 2.5 * y - 1.0).astype(np.float32)
a_ = np.where(np.isinf(s), y, 0).astype(np.uint8)
T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()
sd, zd, yd, ad = T(s, np.float64), T(z, np.float32), T(y, np.uint8), T(a_, np.uint8)
dl, ul = T(sg.delta_grid(s, 100), np.float64), T(sg.logit_grid(100), np.float32)
hist = torch.zeros(N.sweep_hist_words(len(dl), len(ul)), dtype=torch.int64, device="cuda")
ws = N.workspace(N.OP_THRESHOLD_SWEEP, None, None, 0, len(dl), len(ul), device="cuda")
for label, kw in (("ws", {"ws": ws}), ("no-ws", {})):
    for _ in range(3):
        N.noscope_threshold_sweep(1, sd, zd, yd, ad, dl, ul, hist, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(5):
        N.noscope_threshold_sweep(1, sd, zd, yd, ad, dl, ul, hist, **kw)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{label}: events {e0.elapsed_time(e1) / 5:.4f} ms/call, host {(t1 - t0) / 5 * 1e3:.4f} ms/call")
