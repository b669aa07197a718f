"""Parity at BASELINE.json's full size, in the launch configuration bench.py
times: one hour of 640x480 webcam (108,000 frames, 99.5 GB in HBM), blocked
MSE vs t-30, CNN L2C32D32, one noscope_cascade_run over the whole unit.

The oracle recomputes sampled frames one by one (random-access generator):
scores and dispositions bit-exact, small frames byte-exact, logits within
2e-2 — samples include the first frames (forced fires), the boundaries of the
persistent kernel's per-CTA frame ranges (where anchors come from the
previous CTA) and random frames; the label track is checked everywhere
through the label rules (O8) that hold at any size."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import ns, requires_gpu

pytestmark = [pytest.mark.gpu, requires_gpu]

W, H, N, K = 640, 480, 108_000, 30


def test_webcam_hour_sampled_parity():
    nsm = ns()
    from synthgen.gpu import GpuScene, truth_labeller_address
    free, total = torch.cuda.mem_get_info()
    if free < 110e9:
        pytest.skip("needs ~110 GB of free HBM")
    sc = sg.make_scene(sg.SceneSpec(W, H, N, seed=2, stream=0))
    gs = GpuScene(sc)
    pitch = sg.frame_pitch(W, H)
    frames = torch.empty((N, pitch), dtype=torch.uint8, device="cuda")
    for t0 in range(0, N, 4096):
        gs.render(frames[t0:t0 + 4096], t0, min(4096, N - t0))
    lr_w, lr_b = sg.lr_weights(10, 3)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 3)
    delta = 2160.0
    dd = nsm.DD(mode=1, metric=1, grid=10, t_diff_frames=K, t_skip_frames=1, delta_diff=delta,
                lr_weights=torch.from_numpy(lr_w).cuda(), lr_bias=float(lr_b))
    lo, hi = 0.0107, 0.1035
    state = nsm.noscope_stream_state_init(dd)
    route = torch.zeros(N, dtype=torch.uint8, device="cuda")
    logits = torch.full((N,), float("nan"), device="cuda")
    scores = torch.zeros(N, dtype=torch.float64, device="cuda")
    out = nsm.noscope_cascade_run(dd, nsm.Arch(2, 32, 32), nsm.Weights(w), lo, hi, frames, W, H, state,
                                  truth_labeller_address(), gs.truth, route_out=route,
                                  logits_out=logits, scores_out=scores, want_stats=True)
    torch.cuda.synchronize()
    labels = out["labels"].cpu().numpy()
    route = route.cpu().numpy()
    logits = logits.cpu().numpy()
    scores = scores.cpu().numpy()
    del frames
    torch.cuda.empty_cache()

    # ---- label rules everywhere (O8, O7)
    truth = sc.truth
    r = route
    assert np.all(r != O.R_SKIP)                                   # t_skip = 1
    sup = np.flatnonzero(r == O.R_SUPP)
    assert np.array_equal(labels[sup], labels[sup - K])           # mode 1: copy label(t-k)
    assert np.all(labels[r == O.R_NEG] == 0) and np.all(labels[r == O.R_POS] == 1)
    unc = r == O.R_UNC
    assert np.array_equal(labels[unc], truth[unc])                 # stand-in labeller answers
    fired = np.flatnonzero(r >= O.R_NEG)
    assert np.all(np.isinf(scores[:K])) and set(range(K)) <= set(fired.tolist())
    assert out["stats"]["n_fired"] == len(fired)
    zf = logits[fired]
    assert np.array_equal(r[fired] == O.R_NEG, zf < np.float32(lo))
    assert np.array_equal(r[fired] == O.R_POS, zf > np.float32(hi))

    # ---- sampled frames recomputed by the oracle
    rng = np.random.default_rng(0)
    # dd_kernel runs one CTA per SM (148) over contiguous ranges (NOSCOPE_DD_CPS=2
    # gives 296); frames around each boundary take their t-30 anchor from another CTA
    boundary = [int(math.floor(c * N / G)) + d for G, cs in ((148, (1, 2, 77, 147)), (296, (1, 295)))
                for c in cs for d in (-1, 0, 1, 29, 30)]
    samples = sorted(set([0, 1, 29, 30, 31, N - 1] + boundary + rng.integers(K, N, 10).tolist()))
    bg = sg.background(sc.spec)
    fired_samples = []
    for t in samples:
        G = O.downsample(sg.render_frame(sc, t, bg)[None], 50, 50)[0]
        if t >= K:
            A = O.downsample(sg.render_frame(sc, t - K, bg)[None], 50, 50)[0]
            s = O.score_frame(G, A, 1, 10, lr_w, lr_b)
            assert scores[t] == s, (t, scores[t], s)
            assert (r[t] >= O.R_NEG) == (s > delta), t
        if r[t] >= O.R_NEG:
            fired_samples.append((t, G))
    assert fired_samples
    z_o = O.cnn_logits(np.stack([g for _, g in fired_samples]), arch, w)
    z_g = np.array([logits[t] for t, _ in fired_samples])
    assert np.abs(z_g - z_o).max() <= 2e-2
