"""Pins of the oracle's specialized-CNN training (reading R-25):
the hand-written backward pass against torch autograd in fp64 (an independent
implementation of the same network), against central finite differences, the
RMSprop step against torch.optim.RMSprop, and the epoch / early-stopping loop."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import synthgen as sg


def _batch(n, seed, L=2, C=32, D=32):
    rng = np.random.default_rng(seed)
    arch = sg.CnnArch(L, C, D)
    P = O.cnn_params_from_weights(sg.he_normal_weights(arch, seed))
    small = rng.integers(0, 256, (n, 50, 50, 3), dtype=np.uint8)
    t = rng.integers(0, 2, n).astype(np.uint8)
    return arch, P, small, t


def _torch_loss(arch, P, small, t):
    x = torch.tensor(O.normalize_input(small, arch.chan_mean)).permute(0, 3, 1, 2)
    tp = {k: ([torch.tensor(a, requires_grad=True) for a in v] if isinstance(v, list)
              else torch.tensor(v, requires_grad=True)) for k, v in P.items()}
    for l in range(arch.n_conv):
        w = tp["conv_w"][l].permute(0, 3, 1, 2)                       # [Cout, Cin, 3, 3]
        x = F.max_pool2d(F.relu(F.conv2d(x, w, tp["conv_b"][l], padding=1)), 2)
    f = x.permute(0, 2, 3, 1).reshape(x.shape[0], -1)                # (h, w, c) flatten
    h1 = F.relu(f @ tp["fc1_w"].T + tp["fc1_b"])
    z = h1 @ tp["fc2_w"] + tp["fc2_b"][0]
    loss = F.binary_cross_entropy_with_logits(z, torch.tensor(t, dtype=torch.float64))
    loss.backward()
    return loss.item(), z.detach().numpy(), tp


@pytest.mark.parametrize("L", [2, 4])
def test_backward_matches_torch_autograd(L):
    arch, P, small, t = _batch(6, 3, L=L)
    z, st = O.cnn_forward_train(small, arch, P)
    g = O.cnn_backward(z, t, st, P)
    loss_t, z_t, tp = _torch_loss(arch, P, small, t)
    assert np.allclose(z, z_t, rtol=1e-12, atol=1e-12)
    assert abs(O.bce_with_logits(z, t) - loss_t) < 1e-12
    for k in ("fc1_w", "fc1_b", "fc2_w", "fc2_b"):
        assert np.allclose(g[k], tp[k].grad.numpy(), rtol=1e-9, atol=1e-14), k
    for l in range(L):
        assert np.allclose(g["conv_w"][l], tp["conv_w"][l].grad.numpy(), rtol=1e-9, atol=1e-14), l
        assert np.allclose(g["conv_b"][l], tp["conv_b"][l].grad.numpy(), rtol=1e-9, atol=1e-14), l


def test_backward_finite_differences():
    arch, P, small, t = _batch(3, 5)
    z, st = O.cnn_forward_train(small, arch, P)
    g = O.cnn_backward(z, t, st, P)
    rng = np.random.default_rng(0)
    for key, l in [("conv_w", 0), ("conv_w", 1), ("conv_b", 1), ("fc1_w", None), ("fc2_b", None)]:
        arr = P[key][l] if l is not None else P[key]
        gr = g[key][l] if l is not None else g[key]
        for _ in range(3):
            i = tuple(rng.integers(0, s) for s in arr.shape)
            old = arr[i]
            h = 1e-6
            arr[i] = old + h
            lp = O.bce_with_logits(O.cnn_forward_train(small, arch, P)[0], t)
            arr[i] = old - h
            lm = O.bce_with_logits(O.cnn_forward_train(small, arch, P)[0], t)
            arr[i] = old
            assert abs((lp - lm) / (2 * h) - gr[i]) <= 1e-6 * max(1.0, abs(gr[i])), (key, l, i)


def test_rmsprop_matches_torch():
    rng = np.random.default_rng(1)
    p = rng.normal(size=(5, 4))
    v = np.zeros_like(p)
    tp = torch.tensor(p.copy(), requires_grad=True)
    opt = torch.optim.RMSprop([tp], lr=1e-3, alpha=0.9, eps=1e-7)
    P, V = {"fc1_w": p}, {"fc1_w": v}
    for _ in range(4):
        gr = rng.normal(size=p.shape)
        O.rmsprop_step({"conv_w": [], "conv_b": [], "fc1_w": P["fc1_w"], "fc1_b": np.zeros(1),
                        "fc2_w": np.zeros(1), "fc2_b": np.zeros(1)},
                       {"conv_w": [], "conv_b": [], "fc1_w": gr, "fc1_b": np.zeros(1), "fc2_w": np.zeros(1),
                        "fc2_b": np.zeros(1)},
                       {"conv_w": [], "conv_b": [], "fc1_w": V["fc1_w"], "fc1_b": np.zeros(1),
                        "fc2_w": np.zeros(1), "fc2_b": np.zeros(1)}, 1e-3, 0.9, 1e-7)
        tp.grad = torch.tensor(gr)
        opt.step()
    assert np.allclose(P["fc1_w"], tp.detach().numpy(), rtol=1e-13, atol=1e-15)


def _toy(n, seed, learnable=True):
    rng = np.random.default_rng(seed)
    small = rng.integers(40, 90, (n, 50, 50, 3), dtype=np.uint8)
    t = (rng.random(n) < 0.5).astype(np.uint8)
    if learnable:                                           # a bright square iff positive
        for i in np.flatnonzero(t):
            y0, x0 = rng.integers(0, 34, 2)
            small[i, y0:y0 + 16, x0:x0 + 16, :] = 230
    return rng, small, t


@pytest.mark.parametrize("hist,stop", [
    ([(1.0, 0.5)], False),                          # epoch 1 has no predecessor
    ([(1.0, 0.5), (0.9, 0.9)], False),              # train falls, val rises -> continue
    ([(1.0, 0.5), (1.0, 0.4)], False),              # equal is not an increase
    ([(1.0, 0.5), (1.1, 0.4)], True),               # train rises -> stop, even if val improved
    ([(3.0, 1.0), (2.0, 1.0), (2.5, 0.1)], True),
])
def test_stop_rule_is_training_loss_increase(hist, stop):
    """P:474-475 "early stopping if the training loss increases"; "stops early
    when epoch-end training loss exceeds the previous epoch's"."""
    assert O.train_should_stop(hist) is stop


def test_training_learns_and_returns_best_val_epoch():
    """A learnable toy task drives the training loss down over all epochs (no stop);
    the returned parameters are the best cross-validation epoch's."""
    rng, small, t = _toy(96, 2)
    arch = sg.CnnArch(2, 32, 32)
    P0 = O.cnn_params_from_weights(sg.he_normal_weights(arch, 4))
    perms = [rng.permutation(64) for _ in range(3)]
    P, hist = O.cnn_train(small[:64], t[:64], small[64:], t[64:], arch, P0, perms, 16, lr=1e-3)
    assert len(hist) == 3 and hist[2][0] < hist[1][0] < hist[0][0]
    best = min(range(len(hist)), key=lambda e: hist[e][1])
    zb, _ = O.cnn_forward_train(small[64:], arch, P)
    assert abs(O.bce_with_logits(zb, t[64:]) - hist[best][1]) < 1e-12


def test_training_continues_while_val_loss_rises():
    """Cross-validation labels flipped: the training loss keeps falling while the
    validation loss rises every epoch.  The paper's rule keeps training (all 4
    epochs run); the parameters returned are epoch 1's (lowest validation loss)."""
    rng, small, t = _toy(80, 2)
    arch = sg.CnnArch(2, 32, 32)
    P0 = O.cnn_params_from_weights(sg.he_normal_weights(arch, 4))
    perms = [rng.permutation(64) for _ in range(4)]
    P, hist = O.cnn_train(small[:64], t[:64], small[64:], 1 - t[64:], arch, P0, perms, 16, lr=1e-3)
    assert len(hist) == 4
    assert all(hist[e][0] < hist[e - 1][0] and hist[e][1] > hist[e - 1][1] for e in range(1, 4))
    zb, _ = O.cnn_forward_train(small[64:], arch, P)
    assert abs(O.bce_with_logits(zb, 1 - t[64:]) - hist[0][1]) < 1e-12


def test_training_stops_when_training_loss_rises():
    """an oversized learning rate on unlearnable (random) labels makes the
    training loss rise after it first fell -> training stops at that epoch although
    more epochs were allowed; the best cross-validation epoch is returned."""
    rng, small, t = _toy(48, 2, learnable=False)
    arch = sg.CnnArch(2, 32, 32)
    P0 = O.cnn_params_from_weights(sg.he_normal_weights(arch, 4))
    perms = [rng.permutation(32) for _ in range(5)]
    P, hist = O.cnn_train(small[:32], t[:32], small[32:], t[32:], arch, P0, perms, 8, lr=3e-3)
    assert len(hist) == 3 and hist[2][0] > hist[1][0] < hist[0][0]
    best = min(range(3), key=lambda e: hist[e][1])
    zb, _ = O.cnn_forward_train(small[32:], arch, P)
    assert abs(O.bce_with_logits(zb, t[32:]) - hist[best][1]) < 1e-12


def test_training_one_epoch():
    """max_epochs = 1 -> exactly one epoch of updates."""
    rng, small, t = _toy(40, 3)
    arch = sg.CnnArch(2, 32, 32)
    P0 = O.cnn_params_from_weights(sg.he_normal_weights(arch, 5))
    P, hist = O.cnn_train(small[:32], t[:32], small[32:], t[32:], arch, P0, [rng.permutation(32)], 8, lr=1e-3)
    assert len(hist) == 1
