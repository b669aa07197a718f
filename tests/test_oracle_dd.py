"""Pins for the oracle's downsample / MSE / blocked-LR / disposition / compaction /
routing / label functions (O1-O8) against closed forms, library routines and
invariants the paper fixes — none of these re-types the oracle's own formula.

Citations: SPEC.md examples S:197-199 (mse), S:206-208 (blocked_mse)
(dd_score), S:233-235 (dd_step), S:77-79 (preprocess), S:330-332 (classify),
S:479-480 (run_cascade)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg


def rng(seed=0):
    return np.random.default_rng(seed)


# ---------------- O1 downsample ----------------
def test_downsample_identity():
    f = rng().integers(0, 256, (3, 7, 9, 3), dtype=np.uint8)
    assert np.array_equal(O.downsample(f, 7, 9), f)


def test_downsample_constant_frame():
    f = np.full((2, 480, 640, 3), 173, np.uint8)
    assert np.all(O.downsample(f, 50, 50) == 173)


def test_downsample_4x4_to_2x2_block_mean():
    # S:79 "4x4 frame area-averaged to 2x2 -> each output pixel equals mean of its 2x2 block"
    f = np.zeros((1, 4, 4, 3), np.uint8)
    f[0, :2, :2] = [[10, 20, 30], [12, 22, 32]][0]
    f[0, 0, 1] = [14, 24, 34]
    f[0, 2:, 2:] = 200
    g = O.downsample(f, 2, 2)
    assert list(g[0, 0, 0]) == [11, 21, 31]          # (10+14+10+10)/4 = 11
    assert list(g[0, 1, 1]) == [200, 200, 200]
    assert list(g[0, 0, 1]) == [0, 0, 0]


@pytest.mark.parametrize("H,W,h,w", [(100, 100, 50, 50), (150, 200, 50, 50), (8, 12, 4, 3)])
def test_downsample_integer_factor_matches_avg_pool(H, W, h, w):
    f = rng(1).integers(0, 256, (4, H, W, 3), dtype=np.uint8)
    t = torch.from_numpy(f.astype(np.float64)).permute(0, 3, 1, 2)
    kh, kw = H // h, W // w
    s = torch.nn.functional.avg_pool2d(t, (kh, kw)) * (kh * kw)      # exact integer sums
    ref = torch.floor((2 * s + kh * kw) / (2 * kh * kw)).permute(0, 2, 3, 1).numpy()
    assert np.array_equal(O.downsample(f, h, w), ref.astype(np.uint8))


def test_downsample_round_half_up():
    f = np.zeros((1, 2, 1, 3), np.uint8)
    f[0, 0, 0] = [1, 2, 3]
    f[0, 1, 0] = [2, 2, 4]      # means 1.5 -> 2, 2 -> 2, 3.5 -> 4
    assert list(O.downsample(f, 1, 1)[0, 0, 0]) == [2, 2, 4]


def test_downsample_partition_640x480():
    # every source pixel lands in exactly one output cell: a single bright pixel
    # contributes only to its cell, and the cell sums over all outputs scale back
    f = np.zeros((1, 480, 640, 3), np.uint8)
    f[0, 479, 639] = 255
    f[0, 0, 0] = 255
    g = O.downsample(f, 50, 50)
    assert np.count_nonzero(g[..., 0]) == 2
    assert g[0, 49, 49, 0] == round(255 / (9 * 13)) and g[0, 0, 0, 0] == round(255 / (9 * 12))
    with pytest.raises(ValueError):
        O.downsample(f, 481, 50)


# ---------------- O3 MSE ----------------
def test_mse_spec_examples():
    assert O.mse(np.array([0, 0]), np.array([2, 2])) == 4.0
    assert O.mse(np.array([0, 4]), np.array([2, 0])) == 10.0
    a = rng().integers(0, 256, (50, 50, 3))
    assert O.mse(a, a) == 0.0


def test_mse_constant_and_offset():
    p, q = 200, 57
    a = np.full((50, 50, 3), p, np.uint8)
    b = np.full((50, 50, 3), q, np.uint8)
    assert O.mse(a, b) == float((p - q) ** 2)
    base = rng(2).integers(10, 240, (50, 50, 3)).astype(np.uint8)
    for d in (1, 3, 9):
        assert O.mse(base + d, base) == float(d * d)


def test_mse_symmetric_nonneg():
    r = rng(3)
    for _ in range(20):
        a, b = r.integers(0, 256, (2, 11, 13, 3), dtype=np.uint8)
        assert O.mse(a, b) == O.mse(b, a) >= 0.0


def test_blocked_grid1_equals_global():
    a, b = rng(4).integers(0, 256, (2, 50, 50, 3), dtype=np.uint8)
    assert O.blocked_mse(a, b, 1)[0] == O.mse(a, b)


def test_blocked_quadrant():
    # 4x4 frames, grid=2, one quadrant +3 -> one entry 9.0, rest 0
    a = np.full((4, 4, 3), 100, np.uint8)
    b = a.copy()
    b[2:, :2] += 3
    v = O.blocked_mse(a, b, 2)
    assert list(v) == [0.0, 0.0, 9.0, 0.0]


def test_blocked_mean_decomposition():
    r = rng(5)
    for (h, w, g) in [(50, 50, 10), (50, 50, 7), (13, 17, 4)]:
        a, b = r.integers(0, 256, (2, h, w, 3), dtype=np.uint8)
        m = O.blocked_mse(a, b, g)
        sizes = [(r1 - r0) * (c1 - c0) * 3 for (r0, r1) in O.block_bounds(h, g)
                 for (c0, c1) in O.block_bounds(w, g)]
        assert sum(sizes) == h * w * 3
        assert math.isclose(sum(n * v for n, v in zip(sizes, m)) / (h * w * 3), O.mse(a, b),
                            rel_tol=1e-12)


def test_blocked_identical_is_bias():
    # identical frames, blocked metric -> the LR's value at zero features (R-3: logit = b)
    a = rng(6).integers(0, 256, (50, 50, 3), dtype=np.uint8)
    w, b = sg.lr_weights(10, 1)
    assert O.score_frame(a, a, 1, 10, w, b) == -4.0


def test_lr_logit_closed_form():
    assert O.lr_logit(np.array([2.0, 4.0]), np.float32([0.5, 0.25]), 1.0) == 3.0
    # one block differing by d: z = b + w_k * d^2
    a = np.full((50, 50, 3), 80, np.uint8)
    b = a.copy()
    b[5:10, 10:15] += 6                      # block (1, 2) of a 10x10 grid
    w, bias = sg.lr_weights(10, 2)
    z = O.score_frame(b, a, 1, 10, w, bias)
    assert z == float(bias) + float(w[12]) * 36.0


# ---------------- O4 disposition ----------------
def _static_small(n, seed=7):
    f = np.repeat(rng(seed).integers(0, 256, (1, 50, 50, 3), dtype=np.uint8), n, axis=0)
    return f


def test_identical_frames_never_fire():
    small = _static_small(40)
    for mode in (0, 1):
        for delta in (0.0, 1.0, 1e9):
            cfg = O.DDConfig(mode=mode, metric=0, t_diff_frames=5, delta_diff=delta,
                             ref_image=small[0])
            s, d = O.diff_detect(small, cfg)
            fired = np.flatnonzero(d == O.FIRED)
            if mode == 0:
                assert len(fired) == 0
            else:
                assert list(fired) == [0, 1, 2, 3, 4]      # only the forced tau < k


def test_delta_extremes_and_skip_count():
    r = rng(8)
    small = r.integers(0, 256, (100, 50, 50, 3), dtype=np.uint8)
    ref = r.integers(0, 256, (50, 50, 3), dtype=np.uint8)
    cfg = O.DDConfig(mode=0, delta_diff=math.inf, ref_image=ref)
    _, d = O.diff_detect(small, cfg)
    assert np.all(d == O.SUPPRESSED)
    cfg = O.DDConfig(mode=0, delta_diff=-math.inf, ref_image=ref, t_skip_frames=15)
    _, d = O.diff_detect(small, cfg)
    assert (d != O.SKIPPED).sum() == math.ceil(100 / 15)
    assert np.all(d[d != O.SKIPPED] == O.FIRED)


def test_firing_monotone_in_delta():
    r = rng(9)
    small = r.integers(0, 256, (60, 50, 50, 3), dtype=np.uint8)
    prev = None
    for delta in np.linspace(0, 12000, 13):
        cfg = O.DDConfig(mode=1, metric=0, t_diff_frames=3, delta_diff=delta)
        _, d = O.diff_detect(small, cfg)
        cur = set(np.flatnonzero(d == O.FIRED))
        if prev is not None:
            assert cur <= prev
        prev = cur


def test_tie_suppresses():
    a = np.full((1, 50, 50, 3), 10, np.uint8)
    ref = np.full((50, 50, 3), 12, np.uint8)        # MSE exactly 4.0
    _, d = O.diff_detect(a, O.DDConfig(mode=0, delta_diff=4.0, ref_image=ref))
    assert d[0] == O.SUPPRESSED                          # R-4 strict '>'
    _, d = O.diff_detect(a, O.DDConfig(mode=0, delta_diff=np.nextafter(4.0, 0), ref_image=ref))
    assert d[0] == O.FIRED


# ---------------- O5 / O7 / O8 ----------------
def test_compact_matches_flatnonzero():
    d = rng(10).integers(0, 3, 5000).astype(np.uint8)
    assert np.array_equal(O.compact(d), np.flatnonzero(d == 2))


def test_route_spec_examples():
    logit = lambda c: math.log(c / (1 - c))
    assert list(O.route(np.float32([-3, 0, 5]), -math.inf, math.inf)) == [O.R_UNC] * 3
    z = np.float32([logit(0.9)])
    assert O.route(z, logit(0.1), logit(0.8))[0] == O.R_POS
    z = np.float32([-1.25])
    assert O.route(z, -1.25, 3.0)[0] == O.R_UNC                 # c == c_low defers
    assert O.route(np.float32([-1.2500001]), -1.25, 3.0)[0] == O.R_NEG
    with pytest.raises(ValueError):
        O.route(z, 1.0, 0.0)


def test_uncertain_monotone_in_band():
    z = rng(11).normal(0, 2, 2000).astype(np.float32)
    prev = -1
    for wdt in np.linspace(0, 6, 25):
        u = int((O.route(z, -wdt, wdt) == O.R_UNC).sum())
        assert u >= prev
        prev = u


def _tiny_scene(n=300, prevalence=0.3, seed=1):
    sc = sg.make_scene(sg.SceneSpec(50, 50, n, seed=seed, prevalence=prevalence))
    fr = sg.render_frames(sc)[:, :7500].reshape(n, 50, 50, 3)
    return sc, fr


def test_labels_degenerate_passthrough_equals_labeller():
    # S:479 / S:648: no effective DD, thresholds (0,1) -> labels == oracle labels
    sc, fr = _tiny_scene()
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 1)
    cfg = O.DDConfig(mode=0, delta_diff=-math.inf, ref_image=sg.background(sc.spec))
    out = O.cascade(fr, cfg, arch, w, -math.inf, math.inf, sc.truth)
    assert np.array_equal(out["labels"], sc.truth)
    assert np.all(out["route"] == O.R_UNC)


def test_labels_static_video_all_zero():
    # delta = +inf on a static empty video -> predicted all absent, no calls
    small = _static_small(50)
    cfg = O.DDConfig(mode=0, delta_diff=math.inf, ref_image=small[0], t_skip_frames=7)
    s, d = O.diff_detect(small, cfg)
    L = O.resolve_labels(d, np.zeros(50, np.uint8), np.ones(50, np.uint8), 0, 1, 7)
    assert np.all(L == 0)


def test_cascade_partition_and_subset():
    sc, fr = _tiny_scene(seed=3)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 2)
    cfg = O.DDConfig(mode=1, metric=1, grid=10, t_diff_frames=4, t_skip_frames=3,
                     delta_diff=-3.0, lr_w=sg.lr_weights(10, 3)[0], lr_b=-4.0)
    out = O.cascade(fr, cfg, arch, w, -0.5, 0.5, sc.truth)
    r = out["route"]
    counts = [(r == c).sum() for c in range(5)]
    assert sum(counts) == len(r)                                   # S:493 partition
    assert set(np.flatnonzero(r == O.R_UNC)) <= set(out["idx"])    # S:494 subset
    # skipped frames copy their checked frame; mode-1 suppressed copy t-k
    L, d = out["labels"], out["disp"]
    for t in range(len(d)):
        if d[t] == O.SKIPPED:
            assert L[t] == L[t - t % 3]
        elif d[t] == O.SUPPRESSED:
            assert L[t] == L[t - 4]


def test_records_builder():
    s = np.array([5.0, -math.inf, -math.inf, 1.0, math.inf, -math.inf])
    y = np.array([1, 0, 0, 0, 1, 1], np.uint8)
    a = O.build_records(s, y, mode=1, k=2)
    assert list(a) == [0, 1, 1, 0, 0, 1]     # a[3] = y[1], a[5] = y[4]
    a0 = O.build_records(s, y, mode=0, k=2)
    assert list(a0) == [0, 1, 1, 0, 0, 1]
