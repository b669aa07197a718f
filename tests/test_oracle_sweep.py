"""Pins for the oracle's CBO threshold sweep (O9): the cost-model example
(formula P:696), the SPEC 6-frame instance against a
pure-Python brute force that simulates the cascade per triple, random
instances with ties and ±inf, the paper's own greedy procedure
 with readings R-14/R-15, and monotonicity of the uncertain count."""
import math

import numpy as np
import pytest

import oracle as O
import synthgen as sg


def test_cost_model_example():
    # f_s=0.5, f_m=0.2, f_c=0.1, T=(1,10,1000) -> 11.5 per frame
    N = 100
    checked, F, U = 50, 10, 1              # f_s N, f_s f_m N, f_s f_m f_c N
    assert O.cost_ps(checked, F, U, 1, 10, 1000) / N == 11.5
    assert O.cost_ps(0, 0, 0, 1, 10, 1000) == 0                       # f_s = 0
    assert O.cost_ps(N, N, N, 1, 10, 1000) / N == 1011                # f = 1


def _spec6():
    s = np.array([9, 8, 5, 4, 2, 1], np.float64)
    y = np.array([1, 1, 0, 1, 0, 0], np.uint8)
    c = np.array([.95, .9, .6, .55, .2, .1])
    z = np.log(c / (1 - c)).astype(np.float32)
    a = np.zeros(6, np.uint8)                                          # anchor label absent
    delta = np.array([-np.inf, 0.5, 1.5, 3, 4.5, 6.5, 8.5, 9.5], np.float64)
    u = np.unique(np.concatenate([[-np.inf, np.inf], z])).astype(np.float32)
    return s, z, y, a, delta, u


def test_spec_six_frame_instance():
    s, z, y, a, delta, u = _spec6()
    timing = (1, 10, 1000)
    lim = 1                                                             # 1/6 of 6 frames
    T, best = O.sweep(s, z, y, a, delta, u, timing, lim, lim)
    bf = O.sweep_brute_force(s, z, y, a, delta, u, timing, lim, lim)
    assert best == bf and best["feasible"]
    # hand check: fire everything (delta=-inf) costs 6+60+1000*U; the optimum
    # leaves at most one error per side
    assert best["fp"] <= 1 and best["fn"] <= 1


@pytest.mark.parametrize("seed", range(120))
def test_random_instances_equal_brute_force_and_greedy(seed):
    n = 8 + seed % 40
    s, z, y, a, delta, u = sg.random_sweep_records(n, seed)
    timing = [(1, 10, 1000), (5, 7, 11), (0, 1, 1)][seed % 3]
    fp_lim, fn_lim = seed % 4, (seed // 4) % 4
    T, best = O.sweep(s, z, y, a, delta, u, timing, fp_lim, fn_lim)
    bf = O.sweep_brute_force(s, z, y, a, delta, u, timing, fp_lim, fn_lim)
    assert best == bf
    g = O.sweep_greedy_paper(s, z, y, a, delta, u, timing, fp_lim, fn_lim)
    if best["feasible"]:
        assert g is not None and {k: g[k] for k in ("j", "l", "h", "cost", "U")} == \
            {k: best[k] for k in ("j", "l", "h", "cost", "U")}
    else:
        assert g is None


def test_uncertain_count_monotone_in_band():
    # R-18: widening [c_low, c_high] never reduces reference calls
    s, z, y, a, delta, u = sg.random_sweep_records(500, 3)
    T = O.sweep_tables(s, z, y, a, delta, u)
    m = len(u)
    for j in range(len(delta)):
        for l in range(m):
            prev = -1
            for h in range(l, m):
                U = O.triple_counts(T, j, l, h)[3]
                assert U >= prev
                prev = U
            if l > 0:
                for h in range(l, m):
                    assert O.triple_counts(T, j, l - 1, h)[3] >= O.triple_counts(T, j, l, h)[3]


def test_unconstrained_optimum_suppresses_everything():
    # targets (1,1) -> no constraint -> delta above every finite score
    s, z, y, a, delta, u = sg.random_sweep_records(60, 11)
    n = len(s)
    T, best = O.sweep(s, z, y, a, delta, u, (1, 10, 1000), n, n)
    assert best["feasible"] and best["U"] == 0
    assert best["F"] == int((s == np.inf).sum()) + int((s > delta[-1]).sum() - (s == np.inf).sum())


def test_infeasible_reports_best_effort():
    s = np.array([1.0, 2.0], np.float64)
    z = np.float32([0.0, 0.0])
    y = np.array([1, 0], np.uint8)
    a = np.array([0, 1], np.uint8)
    delta = np.array([5.0])                      # nothing fires -> 1 FP + 1 FN forced
    u = np.float32([-1.0, 1.0])
    T, best = O.sweep(s, z, y, a, delta, u, (1, 1, 1), 0, 0)
    assert not best["feasible"] and best["fp"] == 1 and best["fn"] == 1


def test_cbo_search_equals_brute_force_over_pairs():
    """NEXT #2 pin: the CBO's pair search (R-23) picks the same (DD config, CNN,
    triple) as exhaustively simulating the cascade for every pair and triple
    (sweep_brute_force simulates each triple frame by frame)."""
    import synthgen as sg
    rng = np.random.default_rng(7)
    n = 60
    sc = sg.make_scene(sg.SceneSpec(12, 12, n, seed=5, prevalence=0.4, noise_sigma=2))
    small = sg.render_frames(sc)[:, :12 * 12 * 3].reshape(n, 12, 12, 3)
    y = sc.truth[:n].astype(np.uint8)
    ref = sg.background(sc.spec)
    cfgs = [O.DDConfig(mode=0, metric=0, out_w=12, out_h=12, delta_diff=0.0, ref_image=ref),
            O.DDConfig(mode=1, metric=0, out_w=12, out_h=12, t_diff_frames=3, t_skip_frames=2,
                       delta_diff=0.0)]
    grids = []
    for c in cfgs:
        s, _ = O.diff_detect(small, c)
        grids.append(sg.delta_grid(s, 6))
    # two "CNNs" given by their logits: cnn_logits is pinned elsewhere; here the
    # search logic is the object, so the per-arch logits enter through a stub
    z_sets = [rng.normal(0, 1, n) + 2.0 * y, rng.normal(0, 2, n) + 1.0 * y]
    u = np.array([-np.inf, -1.0, 0.0, 0.5, 1.0, 2.0, np.inf])
    t_snn = [40, 15]
    orig = O.cnn_logits
    try:
        it = iter(z_sets)
        O.noscope_oracle.cnn_logits = lambda sm, arch, w: next(it)
        d, c, b = O.noscope_oracle.cbo_search(small, y, cfgs, grids, [(None, None, t) for t in t_snn], u,
                                              5, 1000, 4, 4)
    finally:
        O.noscope_oracle.cnn_logits = orig
    cands = []
    for di, cfg in enumerate(cfgs):
        s, _ = O.diff_detect(small, cfg)
        a = O.build_records(s, y, cfg.mode, cfg.t_diff_frames)
        for ci in range(2):
            bb = O.sweep_brute_force(s, z_sets[ci], y, a, grids[di], u, (5, t_snn[ci], 1000), 4, 4)
            if bb is not None:
                cands.append(((0, 0, bb["cost"], bb["U"], di, ci), di, ci, bb))
    assert cands, "instance must have a feasible pair"
    _, d_bf, c_bf, bb = min(cands, key=lambda x: x[0])
    assert (d, c) == (d_bf, c_bf)
    assert (b["j"], b["l"], b["h"], b["cost"]) == (bb["j"], bb["l"], bb["h"], bb["cost"])
