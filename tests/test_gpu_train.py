"""GPU parity of specialized-CNN training (reading R-25)
against the oracle's fp64 cnn_train: gradients through one RMSprop step in its
linear regime, loss histories and early stopping over epochs, and the export to
inference weights."""
import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import hw3, ns, requires_gpu, scene_frames

pytestmark = [pytest.mark.gpu, requires_gpu]


def _data(n, seed, prevalence=0.5):
    sc, fr = scene_frames(50, 50, n, seed=seed, prevalence=prevalence)
    small = np.zeros((n, 7504), np.uint8)
    small[:, :7500] = fr[:, :7500]
    return small, hw3(fr, 50, 50), sc.truth[:n].astype(np.uint8)


def _flat(P):
    parts = []
    for l in range(len(P["conv_w"])):
        parts += [P["conv_w"][l].ravel(), P["conv_b"][l].ravel()]
    parts += [P["fc1_w"].ravel(), P["fc1_b"].ravel(), P["fc2_w"].ravel(), P["fc2_b"].ravel()]
    return np.concatenate(parts)


@pytest.mark.parametrize("L,C", [(2, 32), (4, 32)])
def test_one_step_gradients(L, C):
    """eps = 1 >> sqrt(v): the step is -lr * g / (sqrt(0.1 g^2) + 1), a smooth function
    of the gradient, so parameter deltas compare the fp32 backward pass with the
    oracle's fp64 one."""
    nsm = ns()
    small, g, y = _data(24, 5)
    arch = sg.CnnArch(L, C, 32)
    w = sg.he_normal_weights(arch, 6)
    A = nsm.Arch(L, C, 32)
    p0 = nsm.params_from_weight_dict(A, w)
    p = p0.clone()
    perm = torch.arange(24, dtype=torch.int32, device="cuda").reshape(1, 24)
    val = torch.arange(4, dtype=torch.int32, device="cuda")
    hist, run = nsm.noscope_cnn_train(A, p, torch.from_numpy(small).cuda(), torch.from_numpy(y).cuda(), perm, val,
                                      batch=24, lr=1.0, rho=0.9, eps=1.0)
    P0 = O.cnn_params_from_weights(w)
    P1, hist_o = O.cnn_train(g, y, g[:4], y[:4], arch, P0, [np.arange(24)], 24, lr=1.0, rho=0.9, eps=1.0)
    d_gpu = (p - p0).cpu().numpy().astype(np.float64)
    d_o = _flat(P1) - _flat(P0)
    scale = np.abs(d_o).max()
    assert np.abs(d_gpu - d_o).max() <= 1e-3 * scale, (np.abs(d_gpu - d_o).max(), scale)
    assert abs(hist[0][0] - hist_o[0][0]) <= 1e-5 * abs(hist_o[0][0])     # loss before the step


def _toy(n, seed, learnable=True):
    """The oracle pins' toy task (tests/test_oracle_train.py::_toy), in the ABI layout."""
    rng = np.random.default_rng(seed)
    g = rng.integers(40, 90, (n, 50, 50, 3), dtype=np.uint8)
    t = (rng.random(n) < 0.5).astype(np.uint8)
    if learnable:
        for i in np.flatnonzero(t):
            y0, x0 = rng.integers(0, 34, 2)
            g[i, y0:y0 + 16, x0:x0 + 16, :] = 230
    small = np.zeros((n, 7504), np.uint8)
    small[:, :7500] = g.reshape(n, -1)
    return rng, small, g, t


def test_training_continues_while_val_loss_rises():
    """stopping follows the TRAINING loss.  Cross-validation labels flipped:
    the validation loss rises every epoch while the training loss falls, so all 4
    epochs run on both sides and the parameters returned are epoch 1's."""
    nsm = ns()
    rng, small, g, t = _toy(80, 2)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 4)
    perms = np.stack([rng.permutation(64) for _ in range(4)]).astype(np.int32)
    lab = t.copy()
    lab[64:] = 1 - lab[64:]
    A = nsm.Arch(2, 32, 32)
    p = nsm.params_from_weight_dict(A, w)
    hist, run = nsm.noscope_cnn_train(A, p, torch.from_numpy(small).cuda(), torch.from_numpy(lab).cuda(),
                                      torch.from_numpy(perms).cuda(),
                                      torch.arange(64, 80, dtype=torch.int32, device="cuda"), batch=16, lr=1e-3)
    _, hist_o = O.cnn_train(g[:64], t[:64], g[64:], lab[64:], arch, O.cnn_params_from_weights(w),
                            list(perms), 16, lr=1e-3)
    assert run == len(hist_o) == 4
    for (a, b), (c, d) in zip(hist, hist_o):
        assert abs(a - c) <= 2e-3 * abs(c) and abs(b - d) <= 2e-3 * abs(d), (hist, hist_o)
    # the returned parameters are epoch 1's (the lowest validation loss)
    Wt = nsm.noscope_cnn_params_to_weights(A, p, nsm.Weights(w))
    z = nsm.noscope_specialized_infer(A, Wt, torch.from_numpy(small[64:]).cuda()).cpu().numpy()
    bce = float(np.mean(np.logaddexp(0, z) - lab[64:] * z))
    assert abs(bce - hist[0][1]) < 0.05 * abs(hist[0][1]) + 0.02      # bf16 inference of the fp32 model


def test_training_stops_when_training_loss_rises():
    """an oversized learning rate on random labels makes the training loss rise
    after it first fell; the GPU stops at that epoch (its own history obeys the rule:
    every earlier epoch did not rise, the last one did) and returns its best
    cross-validation epoch.  (This regime is chaotic, so fp32 and fp64 trajectories
    are compared only through the rule, not value by value.)"""
    nsm = ns()
    rng, small, g, t = _toy(48, 2, learnable=False)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 4)
    perms = np.stack([rng.permutation(32) for _ in range(5)]).astype(np.int32)
    A = nsm.Arch(2, 32, 32)
    p = nsm.params_from_weight_dict(A, w)
    hist, run = nsm.noscope_cnn_train(A, p, torch.from_numpy(small).cuda(), torch.from_numpy(t).cuda(),
                                      torch.from_numpy(perms).cuda(),
                                      torch.arange(32, 48, dtype=torch.int32, device="cuda"), batch=8, lr=3e-3)
    assert run == len(hist) < 5
    tr = [h[0] for h in hist]
    assert tr[-1] > tr[-2] and all(tr[e] <= tr[e - 1] for e in range(1, run - 1))
    _, hist_o = O.cnn_train(g[:32], t[:32], g[32:], t[32:], arch, O.cnn_params_from_weights(w),
                            list(perms), 8, lr=3e-3)
    assert len(hist_o) < 5          # the oracle also stops early on this instance


def test_params_to_weights_rounding():
    nsm = ns()
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 9)
    A = nsm.Arch(2, 32, 32)
    p = nsm.params_from_weight_dict(A, w) * 1.001                        # off the bf16 grid
    out = nsm.noscope_cnn_params_to_weights(A, p, nsm.Weights(sg.zero_weights(arch)))
    n0 = w["conv_w"][0].size
    exp = p[:n0].to(torch.bfloat16).view(torch.int16)
    assert torch.equal(out.conv_w[0].view(-1), exp)
    assert torch.equal(out.conv_b[0], p[n0:n0 + 32])


@pytest.mark.parametrize("L,n_train,batch", [(2, 200, 32), (4, 96, 16)])
def test_graph_replay_equals_plain_launches(L, n_train, batch, monkeypatch):
    """Full mini-batches after the first replay one captured CUDA graph of the step
    (train.cu); the same kernels in the same order, so the parameters and loss
    histories are bit-identical to plain launches (NOSCOPE_TRAIN_GRAPH=0) — with a
    partial last batch (200 = 6 x 32 + 8) that runs outside the graph."""
    nsm = ns()
    n = n_train + 32
    small, g, y = _data(n, 11)
    arch = sg.CnnArch(L, 32, 32)
    A = nsm.Arch(L, 32, 32)
    w = sg.he_normal_weights(arch, 12)
    rng = np.random.default_rng(3)
    perms = torch.from_numpy(np.stack([rng.permutation(n_train) for _ in range(3)]).astype(np.int32)).cuda()
    val = torch.arange(n_train, n, dtype=torch.int32, device="cuda")
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("NOSCOPE_TRAIN_GRAPH", mode)
        p = nsm.params_from_weight_dict(A, w)
        hist, run = nsm.noscope_cnn_train(A, p, torch.from_numpy(small).cuda(), torch.from_numpy(y).cuda(),
                                          perms, val, batch=batch, lr=1e-3)
        out[mode] = (p.cpu().numpy(), hist, run)
    assert out["0"][2] == out["1"][2]
    assert out["0"][1] == out["1"][1]
    assert np.array_equal(out["0"][0].view(np.uint32), out["1"][0].view(np.uint32))
