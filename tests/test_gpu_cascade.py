"""GPU parity for noscope_cascade_run (whole per-frame cascade) against the
oracle's cascade on the same seeded video, including chunked processing of one
unit with carried stream state.  Routing is compared bit-exact: thresholds are
placed in gaps of the oracle logits wider than the measured GPU-oracle logit
deviation, which the test asserts (SURVEY §8(c) "CNN logits" pin)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import dd_pair, hw3, ns, pick_thresholds_in_gaps, requires_gpu, scene_frames

pytestmark = [pytest.mark.gpu, requires_gpu]


def _oracle_logits(small_o, ocfg, arch, w):
    s, d = O.diff_detect(small_o, ocfg)
    idx = O.compact(d)
    return idx, O.cnn_logits(small_o[idx], arch, w)


def _run_cascade(nsm, g, A, W, lo, hi, fr, Wd, Hd, truth, chunks, base=0):
    from synthgen.gpu import truth_labeller_address
    n = fr.shape[0]
    state = nsm.noscope_stream_state_init(g)
    truth_d = torch.from_numpy(truth).cuda()
    labels = np.empty(n, np.uint8)
    route = np.empty(n, np.uint8)
    logits = np.full(n, np.nan, np.float32)
    scores = np.empty(n)
    stats = []
    pos = 0
    for c in chunks:
        f = torch.from_numpy(fr[pos:pos + c]).cuda()
        r_d = torch.zeros(c, dtype=torch.uint8, device="cuda")
        z_d = torch.full((c,), float("nan"), device="cuda")
        s_d = torch.zeros(c, dtype=torch.float64, device="cuda")
        out = nsm.noscope_cascade_run(g, A, W, lo, hi, f, Wd, Hd, state, truth_labeller_address(),
                                      truth_d, seg_offset=pos, frame_index_base=base + pos,
                                      route_out=r_d, logits_out=z_d, scores_out=s_d, want_stats=True)
        torch.cuda.synchronize()
        labels[pos:pos + c] = out["labels"].cpu().numpy()
        route[pos:pos + c] = r_d.cpu().numpy()
        logits[pos:pos + c] = z_d.cpu().numpy()
        scores[pos:pos + c] = s_d.cpu().numpy()
        stats.append(out["stats"])
        pos += c
    return labels, route, logits, scores, stats


def _check(o, labels, route, logits, scores, stats, margin):
    idx = o["idx"]
    dz = np.abs(logits[idx] - o["logits"]).max() if len(idx) else 0.0
    assert dz <= 2e-2
    assert margin > dz, "thresholds not separated from logits by more than the CNN deviation"
    assert np.array_equal(scores, o["score"])
    assert np.array_equal(route, o["route"])
    assert np.array_equal(labels, o["labels"])
    tot = {k: sum(s[k] for s in stats) for k in stats[0]}
    r = o["route"]
    assert tot["n_frames"] == len(r)
    assert tot["n_skipped"] == (r == O.R_SKIP).sum() and tot["n_suppressed"] == (r == O.R_SUPP).sum()
    assert tot["n_neg"] == (r == O.R_NEG).sum() and tot["n_pos"] == (r == O.R_POS).sum()
    assert tot["n_uncertain"] == (r == O.R_UNC).sum()
    assert tot["n_fired"] == len(idx)


def test_tiny_config_cascade():
    """BASELINE configs[0]: 1,000 50x50 frames, global MSE vs reference image,
    2-conv/32-filter CNN, random init weights, fixed thresholds."""
    nsm = ns()
    n = 1000
    sc, fr = scene_frames(50, 50, n, seed=1, prevalence=0.15)
    small = hw3(fr, 50, 50)
    ref = sg.background(sc.spec)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 1)
    ocfg, g = dd_pair(nsm, 0, 0, delta=20.0, ref=ref)
    idx, z = _oracle_logits(small, ocfg, arch, w)
    assert 50 < len(idx) < n
    lo, hi, margin = pick_thresholds_in_gaps(z, 2e-2)
    o = O.cascade(small, ocfg, arch, w, lo, hi, sc.truth)
    assert (o["route"] == O.R_UNC).sum() > 0 and (o["route"] == O.R_NEG).sum() > 0
    res = _run_cascade(nsm, g, nsm.Arch(2, 32, 32), nsm.Weights(w), lo, hi, fr, 50, 50, sc.truth, [n])
    _check(o, *res, margin)


@pytest.mark.parametrize("t_skip,chunks", [(1, [64, 56]), (3, [50, 1, 69]), (1, [120])])
def test_webcam_blocked_lag_chunked(t_skip, chunks):
    nsm = ns()
    n = sum(chunks)
    sc, fr = scene_frames(640, 480, n, seed=2, prevalence=0.9)
    small = O.downsample(hw3(fr, 640, 480), 50, 50)
    lr = sg.lr_weights(10, 3)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 2)
    probe = O.DDConfig(mode=1, metric=1, grid=10, t_diff_frames=7, t_skip_frames=t_skip,
                       delta_diff=0.0, lr_w=lr[0], lr_b=lr[1])
    s_tmp, _ = O.diff_detect(small, probe)
    delta = float(np.quantile(s_tmp[np.isfinite(s_tmp)], 0.6))
    ocfg, g = dd_pair(nsm, 1, 1, k=7, t_skip=t_skip, delta=delta, lr=lr)
    idx, z = _oracle_logits(small, ocfg, arch, w)
    lo, hi, margin = pick_thresholds_in_gaps(z, 2e-2, 0.35, 0.65)
    o = O.cascade(hw3(fr, 640, 480), ocfg, arch, w, lo, hi, sc.truth)
    res = _run_cascade(nsm, g, nsm.Arch(2, 32, 32), nsm.Weights(w), lo, hi, fr, 640, 480, sc.truth,
                       chunks)
    _check(o, *res, margin)


def test_degenerate_passthrough_equals_labeller():
    """delta=-inf, t_skip=1, (c_low, c_high) = (0, 1) -> labels ==
    the reference labeller on every frame."""
    nsm = ns()
    n = 300
    sc, fr = scene_frames(50, 50, n, seed=9, prevalence=0.5)
    ref = sg.background(sc.spec)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 7)
    ocfg, g = dd_pair(nsm, 0, 0, delta=-math.inf, ref=ref)
    labels, route, *_ = _run_cascade(nsm, g, nsm.Arch(2, 32, 32), nsm.Weights(w), -math.inf, math.inf,
                                     fr, 50, 50, sc.truth, [n])
    assert np.array_equal(labels, sc.truth) and np.all(route == O.R_UNC)


def test_cascade_cuda_graph_replay():
    """noscope_cascade_run has no host synchronisation without stats (device
    counts drive the CNN/route kernels), so a chunk can be captured once in a CUDA
    graph and replayed on new frames in the same buffers: identical results to a
    direct call."""
    from synthgen.gpu import truth_labeller_address
    nsm = ns()
    n = 256
    sc, fr = scene_frames(50, 50, 2 * n, seed=17, prevalence=0.3)
    ref = sg.background(sc.spec)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 2)
    _, g = dd_pair(nsm, 0, 0, delta=20.0, ref=ref)
    A, W = nsm.Arch(2, 32, 32), nsm.Weights(w)
    frames = torch.from_numpy(fr[:n]).cuda()
    truth = torch.from_numpy(sc.truth[:n].astype(np.uint8)).cuda()
    state = nsm.noscope_stream_state_init(g)
    ws = nsm.workspace(nsm.OP_CASCADE_RUN, g, A, n)
    bufs = dict(labels=torch.zeros(n, dtype=torch.uint8, device="cuda"),
                route_out=torch.zeros(n, dtype=torch.uint8, device="cuda"),
                logits_out=torch.zeros(n, device="cuda"),
                scores_out=torch.zeros(n, dtype=torch.float64, device="cuda"))
    lo, hi = -0.05, 0.05

    def call():
        nsm.noscope_cascade_run(g, A, W, lo, hi, frames, 50, 50, state, truth_labeller_address(), truth,
                                ws=ws, stream=torch.cuda.current_stream(), **bufs)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()                                   # warm-up (one-time function attributes)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        call()
    # new content in the same buffers, then replay
    frames.copy_(torch.from_numpy(fr[n:]))
    truth.copy_(torch.from_numpy(sc.truth[n:2 * n].astype(np.uint8)))
    graph.replay()
    torch.cuda.synchronize()
    got = {k: v.clone() for k, v in bufs.items()}
    call()
    torch.cuda.synchronize()
    for k in bufs:
        assert torch.equal(got[k], bufs[k]), k
    assert int((got["route_out"] == 4).sum()) > 0
