"""Small invocations of the DD, compaction, routing and cascade kernels for
compute-sanitizer (memcheck / racecheck / synccheck).  usage: python tools/sanitize_small.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen as sg
from paper_1703_02529_b200 import noscope as N
from synthgen.gpu import GpuScene, truth_labeller_address

torch.cuda.set_device(0)
for (W, H, n) in [(640, 480, 40), (101, 77, 300)]:
    sc = sg.make_scene(sg.SceneSpec(W, H, n, seed=3, prevalence=0.5))
    gs = GpuScene(sc)
    fr = torch.empty((n, sg.frame_pitch(W, H)), dtype=torch.uint8, device="cuda")
    gs.render(fr, 0, n)
    out = 50 if W == 640 else 23
    grid = 10 if out == 50 else 4
    lr_w, lr_b = sg.lr_weights(grid, 3)
    for mode in (0, 1):
        for metric in (0, 1):
            dd = N.DD(mode=mode, metric=metric, out_w=out, out_h=out, grid=grid, t_diff_frames=5, t_skip_frames=1,
                      delta_diff=-1.0 if metric else 5.0,
                      ref_image=torch.zeros(out * out * 3, dtype=torch.uint8, device="cuda"),
                      lr_weights=torch.from_numpy(lr_w).cuda(), lr_bias=float(lr_b))
            st = N.noscope_stream_state_init(dd)
            r = N.noscope_diff_detect(dd, fr, W, H, state=st)
            torch.cuda.synchronize()
            print(W, H, mode, metric, "fired", int(r["n_fired"].item()))
d = torch.randint(1, 3, (100003,), dtype=torch.uint8, device="cuda")
idx, cnt = N.noscope_compact_fired(d)
idx2, cnt2 = N.noscope_compact_fired(d.clone(), seg_offset=3, t_skip=4)
z = torch.randn(50001, device="cuda")
r, u, nu = N.noscope_route_logits(-0.5, 0.5, z)
torch.cuda.synchronize()
print("compact", int(cnt.item()), int(cnt2.item()), "route", int(nu.item()))
# the whole cascade on a tiny chunk
n = 300
sc = sg.make_scene(sg.SceneSpec(50, 50, n, seed=1, prevalence=0.4))
gs = GpuScene(sc)
fr = torch.empty((n, 7504), dtype=torch.uint8, device="cuda")
gs.render(fr, 0, n)
dd = N.DD(mode=1, metric=1, grid=10, t_diff_frames=30, t_skip_frames=1, delta_diff=-3.0,
          lr_weights=torch.full((100,), 0.01, device="cuda"), lr_bias=-1.0)
st = N.noscope_stream_state_init(dd)
Wt = N.Weights(sg.he_normal_weights(sg.CnnArch(2, 32, 32), 1))
o = N.noscope_cascade_run(dd, N.Arch(2, 32, 32), Wt, -0.5, 0.5, fr, 50, 50, st, truth_labeller_address(), gs.truth,
                          want_stats=True)
torch.cuda.synchronize()
print("cascade", o["stats"])
# every CNN variant (fused C = 32, conv1-only C = 16 / 64 + generic layers, FC) on a few frames
for L, C, D in [(2, 32, 32), (4, 64, 128), (2, 16, 256), (4, 16, 64)]:
    a = sg.CnnArch(L, C, D)
    zc = N.noscope_specialized_infer(N.Arch(L, C, D), N.Weights(sg.he_normal_weights(a, 2)), fr[:130])
    torch.cuda.synchronize()
    print("cnn", a.name, float(zc.abs().max()))
# threshold sweep (all phases) and the LR fit
s, zz, y, a_, delta, uu = sg.random_sweep_records(3000, 2, n_delta=12, m=10)
T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()
hist = torch.zeros(N.sweep_hist_words(len(delta), len(uu)), dtype=torch.int64, device="cuda")
best, code = N.noscope_threshold_sweep(3, T(s, np.float64), T(zz, np.float32), T(y, np.uint8), T(a_, np.uint8),
                                       T(delta, np.float64), T(uu, np.float32), hist, (1, 10, 1000), 30, 30)
print("sweep", best["j"], best["l"], best["h"], code)
F = torch.rand((500, 8), dtype=torch.float64, device="cuda")
t = (F[:, 0] + 0.3 * torch.rand(500, dtype=torch.float64, device="cuda") > 0.6).to(torch.uint8)
print("lr", N.noscope_lr_fit(F, t))
