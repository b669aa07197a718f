"""Run noscope_specialized_infer on N synthetic 50x50 frames for one arch
(for ncu launch lists / full captures).  Usage: python tools/prof_cnn.py L C D [N] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthgen as sg  # noqa: E402
from paper_1703_02529_b200 import noscope as N  # noqa: E402
from synthgen.gpu import GpuScene  # noqa: E402

L, C, D = (int(x) for x in sys.argv[1:4])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 65536
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
sc = sg.make_scene(sg.SceneSpec(50, 50, n, seed=3, prevalence=0.15))
gs = GpuScene(sc)
small = torch.empty((n, 7504), dtype=torch.uint8, device="cuda")
gs.render(small, 0, n)
arch = sg.CnnArch(L, C, D)
W = N.Weights(sg.he_normal_weights(arch, 3))
A = N.Arch(L, C, D)
ws = N.workspace(N.OP_SPECIALIZED_INFER, None, A, n)
out = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(reps):
    N.noscope_specialized_infer(A, W, small, ws=ws, logits=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    N.noscope_specialized_infer(A, W, small, ws=ws, logits=out)
e1.record()
torch.cuda.synchronize()
print(f"{arch.name} n={n}: {e0.elapsed_time(e1) / reps:.3f} ms/iter")
