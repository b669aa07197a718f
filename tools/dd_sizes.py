"""diff_detect at growing unit sizes (640x480, blocked t-30): where does a launch fail?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_1703_02529_b200 import noscope as N  # noqa: E402
from synthgen.gpu import GpuScene  # noqa: E402
W, H = 640, 480
nmax = int(sys.argv[1]) if len(sys.argv) > 1 else 108000
sc = sg.make_scene(sg.SceneSpec(W, H, nmax, seed=2))
gs = GpuScene(sc)
frames = torch.empty((nmax, sg.frame_pitch(W, H)), dtype=torch.uint8, device="cuda")
for t0 in range(0, nmax, 4096):
    gs.render(frames[t0:t0 + 4096], t0, min(4096, nmax - t0))
lr_w, lr_b = sg.lr_weights(10, 3)
for n in [2000, 8000, 30000, 60000, nmax]:
    for mode in (0, 1):
        dd = N.DD(mode=mode, metric=1, grid=10, t_diff_frames=30, t_skip_frames=1, delta_diff=2160.0,
                  lr_weights=torch.from_numpy(lr_w).cuda(), lr_bias=float(lr_b),
                  ref_image=torch.zeros(7500, dtype=torch.uint8, device="cuda"))
        try:
            r = N.noscope_diff_detect(dd, frames[:n], W, H)
            torch.cuda.synchronize()
            print(n, mode, "ok", int(r["n_fired"].item()))
        except Exception as e:
            print(n, mode, "FAIL", e)
            err = torch.cuda.current_stream()
            break
