"""Degenerate and boundary cases of the whole cascade (noscope_cascade_run) against the
oracle: one-frame units, k larger than the unit (every checked frame a forced fire),
t_skip larger than the unit, delta = +inf (the CNN and routing see zero frames),
identical frames (everything suppressed), single-frame chunks with carried state,
and an empty call.  Labels, routes and scores bit-exact, counts exact."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import dd_pair, hw3, ns, requires_gpu, scene_frames
from test_gpu_cascade import _run_cascade

pytestmark = [pytest.mark.gpu, requires_gpu]

ARCH = sg.CnnArch(2, 32, 32)


def _case(nsm, fr, truth, mode, metric, k, t_skip, delta, lo, hi, chunks, ref=None, lr=None):
    small = hw3(fr, 50, 50)
    ocfg, g = dd_pair(nsm, mode, metric, k=k, t_skip=t_skip, delta=delta, ref=ref, lr=lr)
    w = sg.he_normal_weights(ARCH, 4)
    o = O.cascade(small, ocfg, ARCH, w, lo, hi, truth)
    labels, route, logits, scores, stats = _run_cascade(nsm, g, nsm.Arch(2, 32, 32), nsm.Weights(w), lo, hi, fr,
                                                        50, 50, truth, chunks)
    assert np.array_equal(scores, o["score"])
    assert np.array_equal(route, o["route"])
    assert np.array_equal(labels, o["labels"])
    tot = {q: sum(s[q] for s in stats) for q in stats[0]}
    assert tot["n_fired"] == len(o["idx"]) and tot["n_frames"] == len(fr)
    return o


@pytest.mark.parametrize("mode", [0, 1])
def test_one_frame_unit(mode):
    nsm = ns()
    sc, fr = scene_frames(50, 50, 1, seed=3, prevalence=0.9)
    ref = sg.background(sc.spec)
    # lo = hi = +inf: every fired frame is NEG (z < +inf); mode 1 forces frame 0 to fire
    _case(nsm, fr, sc.truth[:1], mode, 0, 5, 1, 10.0, math.inf, math.inf, [1], ref=ref)


def test_lag_longer_than_unit_all_forced():
    """k = 50 > n = 20: every checked frame has tau < k -> forced fire (R-8); routed
    with (-inf, +inf) so every fired frame takes the reference label."""
    nsm = ns()
    sc, fr = scene_frames(50, 50, 20, seed=4, prevalence=0.5)
    o = _case(nsm, fr, sc.truth[:20], 1, 0, 50, 3, 1e9, -math.inf, math.inf, [20])
    assert np.all(o["disp"][::3] == O.FIRED)


def test_skip_longer_than_unit():
    nsm = ns()
    sc, fr = scene_frames(50, 50, 30, seed=5, prevalence=0.5)
    ref = sg.background(sc.spec)
    o = _case(nsm, fr, sc.truth[:30], 0, 0, 1, 100, -math.inf, -math.inf, math.inf, [30], ref=ref)
    assert (o["disp"] != O.SKIPPED).sum() == 1


@pytest.mark.parametrize("mode", [0, 1])
def test_nothing_fires(mode):
    """delta = +inf: compaction yields 0 frames, the CNN and routing run on an empty
    device count, labels follow the not-fired rules only."""
    nsm = ns()
    sc, fr = scene_frames(50, 50, 200, seed=6, prevalence=0.5)
    ref = sg.background(sc.spec)
    o = _case(nsm, fr, sc.truth[:200], mode, 0, 4, 2, math.inf, -0.5, 0.5, [200], ref=ref)
    assert len(o["idx"]) == (2 if mode == 1 else 0)     # mode 1: the forced fires of tau < k


def test_identical_frames_all_suppressed():
    nsm = ns()
    sc, fr = scene_frames(50, 50, 1, seed=7, prevalence=0.0, sigma=0)
    fr = np.repeat(fr, 150, axis=0)
    lr = sg.lr_weights(10, 1)
    o = _case(nsm, fr, np.zeros(150, np.uint8), 1, 1, 3, 1, -3.9, -0.5, 0.5, [150], lr=lr)
    assert (o["disp"] == O.FIRED).sum() == 3                  # only the forced tau < k


def test_single_frame_chunks_with_state():
    nsm = ns()
    n = 37
    sc, fr = scene_frames(50, 50, n, seed=8, prevalence=0.6)
    lr = sg.lr_weights(10, 2)
    _case(nsm, fr, sc.truth[:n], 1, 1, 5, 3, -3.5, -math.inf, math.inf, [1] * n, lr=lr)


def test_empty_call():
    nsm = ns()
    sc, fr = scene_frames(50, 50, 1, seed=9)
    _, g = dd_pair(nsm, 0, 0, ref=sg.background(sc.spec))
    from synthgen.gpu import truth_labeller_address
    state = nsm.noscope_stream_state_init(g)
    w = sg.he_normal_weights(ARCH, 1)
    out = nsm.noscope_cascade_run(g, nsm.Arch(2, 32, 32), nsm.Weights(w), -1.0, 1.0,
                                  torch.zeros((0, 7504), dtype=torch.uint8, device="cuda"), 50, 50, state,
                                  truth_labeller_address(), torch.zeros(1, dtype=torch.uint8, device="cuda"),
                                  want_stats=True)
    torch.cuda.synchronize()
    assert out["stats"]["n_frames"] == 0 and out["stats"]["n_fired"] == 0
