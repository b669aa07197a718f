"""Pins of the oracle's DD fitting steps: reference image
(SPEC S:134-142), block features (O3 per frame), logistic-regression
fit.  Each pin checks against something
other than the oracle's own formula: SPEC's worked examples, exact rational
arithmetic, an analytic optimum, and scipy's general-purpose minimiser."""
import math
from fractions import Fraction

import numpy as np
import pytest
from scipy.optimize import minimize

import oracle as O


# ------------------------------------------------------------ reference image
def test_reference_identical_negatives():
    f = np.random.default_rng(0).integers(0, 256, (7, 5, 3), dtype=np.uint8)
    small = np.stack([f] * 4)
    assert np.array_equal(O.reference_image(small, np.zeros(4, np.uint8)), f)


def test_reference_spec_examples_and_half_up():
    a = np.full((1, 2, 2, 3), 10, np.uint8)
    assert np.all(O.reference_image(np.concatenate([a, a + 10]), np.array([0, 0])) == 15)
    assert np.all(O.reference_image(np.concatenate([a, a + 1]), np.array([0, 0])) == 11)   # 10.5 -> 11
    three = np.concatenate([a, a + 1, a + 1, a + 200])
    assert np.all(O.reference_image(three, np.array([0, 0, 0, 1])) == 11)   # 32/3; positive ignored


def test_reference_no_negative_raises():
    with pytest.raises(ValueError):
        O.reference_image(np.zeros((3, 2, 2, 3), np.uint8), np.ones(3, np.uint8))


def test_reference_brute_force_rational():
    rng = np.random.default_rng(1)
    small = rng.integers(0, 256, (9, 4, 3, 3), dtype=np.uint8)
    lab = rng.integers(0, 2, 9).astype(np.uint8)
    lab[0] = 0
    ref = O.reference_image(small, lab)
    neg = [i for i in range(9) if lab[i] == 0]
    for y in range(4):
        for x in range(3):
            for c in range(3):
                mean = Fraction(sum(int(small[i, y, x, c]) for i in neg), len(neg))
                assert ref[y, x, c] == math.floor(mean + Fraction(1, 2))


# ------------------------------------------------------------ block features
def test_block_features_modes():
    rng = np.random.default_rng(2)
    small = rng.integers(0, 256, (6, 10, 10, 3), dtype=np.uint8)
    ref = rng.integers(0, 256, (10, 10, 3), dtype=np.uint8)
    f0 = O.block_features(small, 3, 0, ref=ref)
    for i in range(6):
        assert np.array_equal(f0[i], O.blocked_mse(small[i], ref, 3))
    f1 = O.block_features(small, 2, 1, k=2)
    assert np.isnan(f1[:2]).all()
    for i in range(2, 6):
        assert np.array_equal(f1[i], O.blocked_mse(small[i], small[i - 2], 2))
    g1 = O.block_features(small, 1, 0, ref=ref)                   # grid 1 = global MSE
    assert np.allclose(g1[:, 0], [O.mse(small[i], ref) for i in range(6)], rtol=0, atol=0)


# ------------------------------------------------------------ LR fit
def test_lr_separable_block_dominates():
    rng = np.random.default_rng(3)
    n, d = 400, 6
    t = (rng.random(n) < 0.4).astype(np.uint8)
    F = rng.gamma(2.0, 50.0, (n, d))
    F[:, 3] = 100.0 + 500.0 * t + rng.random(n)                   # block 3 alone separates
    info = {}
    w, b = O.lr_fit(F, t, info=info)                              # l2 = 1/n: a minimiser exists
    assert info["grad_inf"] <= 1e-9
    pred = (F @ w + b) > 0
    assert (pred == t.astype(bool)).all()
    w_std = np.abs(w * F.std(axis=0))
    assert np.argmax(w_std) == 3 and w_std[3] > 3 * np.delete(w_std, 3).max()


def test_lr_constant_features_analytic_optimum():
    t = np.array([1] * 30 + [0] * 70, np.uint8)
    w, b = O.lr_fit(np.zeros((100, 4)), t)
    assert np.all(w == 0)
    assert abs(b - math.log(0.3 / 0.7)) < 1e-9


def test_lr_column_scaling_invariant():
    rng = np.random.default_rng(4)
    F = rng.gamma(2.0, 10.0, (300, 5))
    t = (F[:, 0] + F[:, 2] + rng.normal(0, 5, 300) > 40).astype(np.uint8)
    w, b = O.lr_fit(F, t, l2=1e-3)
    F2 = F.copy()
    F2[:, 1] *= 10.0
    w2, b2 = O.lr_fit(F2, t, l2=1e-3)
    assert np.allclose(F @ w + b, F2 @ w2 + b2, rtol=1e-9, atol=1e-9)
    assert np.array_equal((F @ w + b) > 0, (F2 @ w2 + b2) > 0)


def _zspace(F, w, b):
    sd, mu = F.std(axis=0), F.mean(axis=0)
    return np.concatenate([w * sd, [b + np.sum(w * mu)]])


def _zobj(F, t, l2):
    sd, mu, d = F.std(axis=0), F.mean(axis=0), F.shape[1]

    def obj(v):          # parameters in the z-scored space, mapped to raw for lr_loss
        ws, bs = v[:d], v[d]
        return O.lr_loss(F, t, ws / sd, bs - np.sum(ws * mu / sd), l2)
    return obj


@pytest.mark.parametrize("l2", [0.05, 1e-3])
def test_lr_fit_is_scipy_minimiser(l2):
    """l2 > 0: J is strongly convex, so the fit must be the minimiser scipy finds on
    lr_loss by finite-difference BFGS (no shared gradient or Hessian code: a sign
    error, a dropped term or a wrong unscaling in lr_fit would miss it)."""
    rng = np.random.default_rng(5)
    n, d = 200, 3
    F = rng.normal(0, 1, (n, d)) * [1.0, 3.0, 0.5] + [2.0, -1.0, 0.0]
    t = (F @ [1.0, -0.5, 2.0] + rng.normal(0, 1.5, n) > 1.0).astype(np.uint8)
    w, b = O.lr_fit(F, t, l2=l2)
    obj = _zobj(F, t, l2)
    res = minimize(obj, np.zeros(d + 1), method="BFGS", options={"gtol": 1e-11})
    v = _zspace(F, w, b)
    assert np.allclose(v, res.x, atol=2e-6), (v, res.x)
    assert obj(v) <= res.fun + 1e-12


def test_lr_fit_stationary_by_finite_differences():
    """Central differences of lr_loss (the objective written on raw parameters) vanish
    at the returned point — a check that shares nothing with lr_fit's gradient."""
    rng = np.random.default_rng(6)
    n, d, l2 = 500, 5, 2e-3
    F = rng.gamma(2.0, 30.0, (n, d))
    t = (F[:, 1] - F[:, 4] + rng.normal(0, 20, n) > 0).astype(np.uint8)
    w, b = O.lr_fit(F, t, l2=l2)
    obj = _zobj(F, t, l2)
    v = _zspace(F, w, b)
    h = 1e-6
    g = np.array([(obj(v + h * e) - obj(v - h * e)) / (2 * h) for e in np.eye(d + 1)])
    assert np.max(np.abs(g)) < 1e-7, g


def test_lr_fit_converges_in_few_newton_steps():
    rng = np.random.default_rng(7)
    F = rng.normal(0, 1, (2000, 20))
    t = (F[:, :3].sum(axis=1) + rng.normal(0, 1, 2000) > 0).astype(np.uint8)
    info = {}
    O.lr_fit(F, t, l2=1e-3, info=info)
    assert info["grad_inf"] <= 1e-9 and info["iters"] <= 15


def test_lr_errors():
    with pytest.raises(ValueError):
        O.lr_fit(np.ones((5, 2)), np.zeros(5, np.uint8))
    with pytest.raises(ValueError):
        O.lr_fit(np.ones((1, 2)), np.ones(1, np.uint8))
    with pytest.raises(ValueError):
        O.lr_fit(np.ones((4, 2)), np.array([0, 1, 0, 1], np.uint8), l2=0.0)
