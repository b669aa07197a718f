"""Time the whole threshold sweep on a tiny record set (phase 2 — tables + the
(delta, c_low, c_high) evaluation — dominates) at the bench's grid size, to A/B
the phase-2 kernels (NOSCOPE_LIB selects the library)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_1703_02529_b200 import noscope as N  # noqa: E402
M = 4096
g = torch.Generator(device="cuda").manual_seed(4)
y = (torch.rand(M, device="cuda", generator=g) < 0.15).to(torch.uint8)
s = torch.empty(M, dtype=torch.float64, device="cuda").exponential_(0.05, generator=g) + 40.0 * y
z = (torch.randn(M, device="cuda", generator=g) + 2.5 * y - 1.0).float()
a = torch.zeros_like(y)
for grid in (100, 400, 1000):
    dl = torch.from_numpy(sg.delta_grid(s.cpu().numpy(), grid)).cuda()
    ul = torch.from_numpy(sg.logit_grid(grid)).cuda()
    hist = torch.zeros(N.sweep_hist_words(len(dl), len(ul)), dtype=torch.int64, device="cuda")
    N.noscope_threshold_sweep(1, s, z, y, a, dl, ul, hist)
    for _ in range(5):
        best = N.noscope_threshold_sweep(2, None, None, None, None, dl, ul, hist, timing=(1, 20, 3000),
                                         fp_limit=M // 100, fn_limit=M // 100)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        N.noscope_threshold_sweep(2, None, None, None, None, dl, ul, hist, timing=(1, 20, 3000),
                                  fp_limit=M // 100, fn_limit=M // 100)
    e1.record()
    torch.cuda.synchronize()
    print(f"grid {grid}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us/sweep  best={best}")
