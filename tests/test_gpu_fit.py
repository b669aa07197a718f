"""GPU parity of the DD fitting steps against the oracle:
reference image (bit-exact), per-frame block features (bit-exact fp64: the same
integer SSD divided by the same count), and the blocked-LR fit (fp64 GD; only the
summation order differs -> 1e-9 relative)."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import dd_pair, hw3, ns, requires_gpu, scene_frames

pytestmark = [pytest.mark.gpu, requires_gpu]


def _small(n, seed, prevalence=0.3, W=50, H=50):
    sc, fr = scene_frames(W, H, n, seed=seed, prevalence=prevalence)
    pitch = (W * H * 3 + 15) // 16 * 16
    small = np.zeros((n, pitch), np.uint8)
    small[:, :W * H * 3] = fr[:, :W * H * 3]
    return sc, small, hw3(fr, W, H)


@pytest.mark.parametrize("n", [1, 37, 3001])
def test_reference_image_bit_exact(n):
    nsm = ns()
    sc, small, g = _small(n, 21)
    lab = sc.truth[:n].astype(np.uint8)
    lab[0] = 0
    ref = nsm.noscope_reference_image(torch.from_numpy(small).cuda(), torch.from_numpy(lab).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(ref.cpu().numpy().reshape(50, 50, 3), O.reference_image(g, lab))


def test_reference_image_ties_and_no_negative():
    nsm = ns()
    pitch = 7504
    small = np.zeros((4, pitch), np.uint8)
    small[0, :7500], small[1, :7500], small[2, :7500], small[3, :7500] = 10, 11, 250, 7
    lab = np.array([0, 0, 1, 1], np.uint8)
    ref = nsm.noscope_reference_image(torch.from_numpy(small).cuda(), torch.from_numpy(lab).cuda())
    assert np.all(ref.cpu().numpy() == 11)                        # 10.5 rounds half up
    with pytest.raises(nsm.NoScopeError) as e:
        nsm.noscope_reference_image(torch.from_numpy(small).cuda(), torch.ones(4, dtype=torch.uint8).cuda())
    assert e.value.code == 6


@pytest.mark.parametrize("mode,grid,k", [(0, 10, 0), (1, 7, 3), (1, 16, 30), (0, 1, 0)])
def test_block_features_bit_exact(mode, grid, k):
    nsm = ns()
    n = 97
    sc, small, g = _small(n, 22)
    ref = O.reference_image(g, sc.truth[:n]) if mode == 0 else None
    _, dd = dd_pair(nsm, mode, 1, grid=grid, k=max(k, 1), ref=ref, lr=(np.ones(grid * grid, np.float32), 0.0))
    f = nsm.noscope_block_features(dd, torch.from_numpy(small).cuda())
    torch.cuda.synchronize()
    got = f.cpu().numpy()
    exp = O.block_features(g, grid, mode, ref=ref, k=k)
    assert np.array_equal(np.isnan(got), np.isnan(exp))
    ok = ~np.isnan(exp)
    assert np.array_equal(got[ok], exp[ok])


def _zspace(F, w, b):
    sd, mu = F.std(axis=0), F.mean(axis=0)
    sd = np.where(sd > 0, sd, 1.0)
    return np.concatenate([w * sd, [b + np.sum(w * mu)]])


def _minimiser_bound(F, t, v, l2, tol):
    """Both fits stop at max|grad J| <= tol; near the unique minimiser v*, v - v* =
    H^{-1} g + O(|g|^2), so two such points differ by at most ||H^{-1}||_inf * 2 tol.
    H is J's Hessian at the oracle's point (z-scored space)."""
    sd, mu = F.std(axis=0), F.mean(axis=0)
    sd = np.where(sd > 0, sd, 1.0)
    X1 = np.hstack([(F - mu) / sd, np.ones((len(F), 1))])
    p = 1.0 / (1.0 + np.exp(-(X1 @ v)))
    H = (X1 * (p * (1 - p))[:, None]).T @ X1 / len(F) + np.diag([l2] * F.shape[1] + [0.0])
    return np.abs(np.linalg.inv(H)).sum(axis=1).max() * 2 * tol


def _compare_fits(F, t, l2, w, b, info, tol=1e-9):
    info_o = {}
    w_o, b_o = O.lr_fit(F, t, l2=l2, tol=tol, info=info_o)
    v, v_o = _zspace(F, w, b), _zspace(F, w_o, b_o)
    bound = _minimiser_bound(F, t, v_o, l2, tol)
    assert info["grad_inf"] <= tol and info_o["grad_inf"] <= tol, (info, info_o)
    assert np.abs(v - v_o).max() <= bound + 1e-12 * np.abs(v_o).max(), (np.abs(v - v_o).max(), bound)
    return w_o, b_o


def test_lr_fit_matches_oracle_on_scene_features():
    """Mode-1 training set as the paper builds it: block MSEs vs frame t-k,
    target = label(t) != label(t-k); GPU features feed the GPU fit.  Both sides
    return the minimiser of the same strictly convex objective to max|grad| <= 1e-9."""
    nsm = ns()
    n, k, grid = 2000, 15, 10
    sc, small, g = _small(n, 23, prevalence=0.4)
    _, dd = dd_pair(nsm, 1, 1, grid=grid, k=k, lr=(np.ones(grid * grid, np.float32), 0.0))
    feats = nsm.noscope_block_features(dd, torch.from_numpy(small).cuda())[k:].contiguous()
    y = sc.truth[:n].astype(np.uint8)
    t = (y[k:] != y[:-k]).astype(np.uint8)
    assert 0 < t.sum() < len(t)
    info = {}
    w, b = nsm.noscope_lr_fit(feats, torch.from_numpy(t).cuda(), l2=1e-3, info=info)
    F = feats.cpu().numpy()
    _compare_fits(F, t, 1e-3, w, b, info)
    # the fitted model separates better than chance on its training set
    acc = ((F @ w + b > 0) == t.astype(bool)).mean()
    assert acc > max(t.mean(), 1 - t.mean())
    # deterministic: a second fit is bitwise identical
    w2, b2 = nsm.noscope_lr_fit(feats, torch.from_numpy(t).cuda(), l2=1e-3)
    assert np.array_equal(w, w2) and b == b2


@pytest.mark.parametrize("n,d", [(4099, 6), (70001, 100)])
def test_lr_fit_separable_and_errors(n, d):
    """A separable set (block 3 decides) at the default l2 = 1/n, incl. a ragged
    multi-CTA size with the webcam grid's d = 100."""
    nsm = ns()
    rng = np.random.default_rng(3)
    t = (rng.random(n) < 0.4).astype(np.uint8)
    F = rng.gamma(2.0, 50.0, (n, d))
    F[:, 3] = 100.0 + 500.0 * t + rng.random(n)
    Fd, td = torch.from_numpy(F).cuda(), torch.from_numpy(t).cuda()
    info = {}
    w, b = nsm.noscope_lr_fit(Fd, td, info=info)
    _compare_fits(F, t, 1.0 / n, w, b, info)
    assert ((F @ w + b > 0) == t.astype(bool)).all()
    with pytest.raises(nsm.NoScopeError):
        nsm.noscope_lr_fit(Fd, torch.zeros(n, dtype=torch.uint8).cuda())   # one class
    Fn = Fd.clone()
    Fn[5, 2] = float("nan")
    with pytest.raises(nsm.NoScopeError):
        nsm.noscope_lr_fit(Fn, td)


def test_lr_fit_constant_features():
    """constant features -> w = 0, b = logit(prevalence)."""
    nsm = ns()
    t = np.array([1] * 300 + [0] * 700, np.uint8)
    w, b = nsm.noscope_lr_fit(torch.full((1000, 4), 3.0, dtype=torch.float64, device="cuda"),
                              torch.from_numpy(t).cuda())
    assert np.all(w == 0) and abs(b - np.log(0.3 / 0.7)) < 1e-9


def test_fitted_weights_drive_the_dd():
    """The fit's raw-feature output plugs into noscope_dd_config (fp32 weights)."""
    nsm = ns()
    n, k, grid = 600, 5, 10
    sc, small, g = _small(n, 24, prevalence=0.4)
    _, dd = dd_pair(nsm, 1, 1, grid=grid, k=k, lr=(np.ones(grid * grid, np.float32), 0.0))
    feats = nsm.noscope_block_features(dd, torch.from_numpy(small).cuda())[k:].contiguous()
    y = sc.truth[:n].astype(np.uint8)
    t = torch.from_numpy((y[k:] != y[:-k]).astype(np.uint8)).cuda()
    w, b = nsm.noscope_lr_fit(feats, t, l2=1e-3)
    F = feats.cpu().numpy()
    z_fit = F @ w + b
    w32, b32 = w.astype(np.float32), np.float32(b)
    z_dd = np.array([O.lr_logit(F[i], w32, b32) for i in range(len(F))])
    assert np.allclose(z_dd, z_fit, rtol=1e-4, atol=1e-3)
