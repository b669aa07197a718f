"""Time noscope_cnn_train like bench.py's extras.next_rows.cnn_train: L2C32D32,
8,192 frames x 2 epochs, batch 64.  usage: python tools/time_train.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_1703_02529_b200 import noscope as N  # noqa: E402
from synthgen.gpu import GpuScene  # noqa: E402
n = 65536
sc = sg.make_scene(sg.SceneSpec(50, 50, n, seed=3, prevalence=0.15))
gs = GpuScene(sc)
small = torch.empty((n, 7504), dtype=torch.uint8, device="cuda")
gs.render(small, 0, n)
y = gs.truth[:n].contiguous()
arch = sg.CnnArch(2, 32, 32)
A = N.Arch(2, 32, 32)
nt, ep = 8192, 2
p = N.params_from_weight_dict(A, sg.he_normal_weights(arch, 3))
perms = torch.stack([torch.randperm(nt, device="cuda") for _ in range(ep)]).to(torch.int32)
val = torch.arange(nt, nt + 1024, dtype=torch.int32, device="cuda")
N.noscope_cnn_train(A, p.clone(), small, y, perms[:1, :128].contiguous(), val[:64], batch=64)
torch.cuda.synchronize()
t0 = time.perf_counter()
hist, run = N.noscope_cnn_train(A, p, small, y, perms, val, batch=64)
dt = time.perf_counter() - t0
print(f"train: {run} epochs of {nt} frames in {dt:.3f} s = {nt * run / dt:.0f} frames/s; history {hist}")
