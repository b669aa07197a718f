"""Run the NEXT-row kernels once on 65,536 50x50 frames (for ncu launch lists)."""
import os, sys
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
for _ in range(2):
    ref = N.noscope_reference_image(small, y)
    dd = N.DD(mode=1, metric=1, grid=10, t_diff_frames=30, lr_weights=torch.ones(100, device="cuda"))
    f = N.noscope_block_features(dd, small)
    F = f[30:].contiguous()
    t = (y[30:] != y[:-30]).to(torch.uint8).contiguous()
    N.noscope_lr_fit(F, t, 5)
    N.noscope_eval_labels(y, y.roll(3))
torch.cuda.synchronize()
print("ok")
