"""Scale points of the compaction (H4) and routing (H6) kernels: 2^30 dispositions,
2^28 logits.  usage: python tools/prof_scan.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_02529_b200 import noscope as N


def t_ms(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


g = torch.Generator(device="cuda").manual_seed(4)
fracs = [float(x) for x in sys.argv[1:]] or [0.15, 0.5]
for frac in fracs:
    NC = 1 << 30
    d = torch.where(torch.rand(NC, device="cuda", generator=g) < frac, torch.full((), 2, dtype=torch.uint8, device="cuda"),
                    torch.full((), 1, dtype=torch.uint8, device="cuda"))
    nf = int((d == 2).sum())
    ws = torch.empty(N.lib().noscope_compact_workspace_bytes(NC), dtype=torch.uint8, device="cuda")
    out = (torch.empty(NC, dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int64, device="cuda"))
    mss = sorted(t_ms(lambda: N.noscope_compact_fired(d, ws=ws, out=out)) for _ in range(5))
    ms = mss[2]
    byt = NC + 4 * nf
    print(f"compaction 2^30 fired {frac}: median {ms:.3f} ms (min {mss[0]:.3f})  {byt / ms / 1e6:.1f} GB/s")
    del d, ws, out
NR = 1 << 28
z = torch.randn(NR, device="cuda", generator=g)
nu = int(((z >= -0.5) & (z <= 0.5)).sum())
ws = torch.empty(N.lib().noscope_route_workspace_bytes(NR), dtype=torch.uint8, device="cuda")
out = (torch.empty(NR, dtype=torch.uint8, device="cuda"), torch.empty(NR, dtype=torch.int32, device="cuda"),
       torch.zeros(1, dtype=torch.int64, device="cuda"))
ms = t_ms(lambda: N.noscope_route_logits(-0.5, 0.5, z, ws=ws, out=out))
byt = 5 * NR + 4 * nu
print(f"routing 2^28: {ms:.3f} ms  {byt / ms / 1e6:.1f} GB/s")
