"""Run the threshold sweep's histogram phase on N synthetic records (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_1703_02529_b200 import noscope as N  # noqa: E402
M = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
g = torch.Generator(device="cuda").manual_seed(4)
y = (torch.rand(M, device="cuda", generator=g) < 0.15).to(torch.uint8)
s = torch.empty(M, dtype=torch.float64, device="cuda").exponential_(0.05, generator=g) + 40.0 * y
s[torch.rand(M, device="cuda", generator=g) < 0.05] = -float("inf")
z = (torch.randn(M, device="cuda", generator=g) + 2.5 * y - 1.0).float()
a = torch.where(torch.isinf(s), y, torch.zeros_like(y))
dl = torch.from_numpy(sg.delta_grid(s[:100000].cpu().numpy(), 100)).cuda()
ul = torch.from_numpy(sg.logit_grid(100)).cuda()
hist = torch.zeros(N.sweep_hist_words(len(dl), len(ul)), dtype=torch.int64, device="cuda")
for _ in range(3):
    N.noscope_threshold_sweep(1, s, z, y, a, dl, ul, hist)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
N.noscope_threshold_sweep(1, s, z, y, a, dl, ul, hist)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"sweep_hist {M} records: {ms:.3f} ms, {M * 14 / ms / 1e6:.1f} GB/s")
