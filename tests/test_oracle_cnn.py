"""Pins for the oracle's specialized CNN (O6): closed forms on special weights
(S:296-304), the normalisation examples, and an independent re-derivation
of the layer algebra with torch's CPU fp64 conv2d / max_pool2d / linear on the same
bf16-rounded tensors (a library routine, not the oracle's per-tap matmul loop)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg


def test_bf16_round_matches_torch():
    x = np.random.default_rng(0).normal(0, 3, 20000).astype(np.float32)
    x = np.concatenate([x, np.float32([1.0, -1.0, 0.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8, 255.5])])
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.bf16_round(x.astype(np.float64)), ref)


def test_normalize_examples():
    g = np.array([[[127, 128, 255]], [[0, 64, 200]]], np.uint8)
    x = O.normalize_input(g, (127.0, 128.0, 127.5))
    assert x[0, 0, 0] == 0.0 and x[0, 0, 1] == 0.0        # pixel == mean -> 0
    assert x[0, 0, 2] == 1.0                              # 255, mean 127.5 -> 1.0
    assert np.all(np.abs(x) <= 1.0)
    assert O.normalize_input(np.array([0], np.uint8), (127.5,))[0] == -1.0


def test_zero_weights_logit_zero():
    for arch in sg.ARCH_GRID[:2]:
        w = sg.zero_weights(arch)
        small = np.random.default_rng(1).integers(0, 256, (3, 50, 50, 3), dtype=np.uint8)
        z = O.cnn_logits(small, arch, w)
        assert np.all(z == 0.0) and np.all(O.sigmoid(z) == 0.5)


def test_bias_ln3_gives_075():
    arch = sg.CnnArch(2, 32, 32)
    w = sg.zero_weights(arch)
    w["fc2_b"] = np.float32([math.log(3.0)])
    z = O.cnn_logits(np.zeros((2, 50, 50, 3), np.uint8), arch, w)
    assert np.allclose(O.sigmoid(z), 0.75, atol=1e-7)


def test_center_tap_identity_passthrough():
    # conv1 = centre-tap identity on 3 channels, conv2 = centre-tap identity on
    # those 3; FC1 picks one feature: z equals that pooled, normalised pixel.
    arch = sg.CnnArch(2, 32, 32)
    w = sg.zero_weights(arch)
    one = sg.bf16_round_f32(np.float32([1.0]))[0]
    for c in range(3):
        w["conv_w"][0][c, 1, 1, c] = one
        w["conv_w"][1][c, 1, 1, c] = one
    C2 = 64
    feat = (3 * 12 + 5) * C2 + 1          # (h=3, w=5, c=1) in (h, w, c) order
    w["fc1_w"][0, feat] = one
    w["fc2_w"][0] = one
    g = np.random.default_rng(2).integers(0, 256, (4, 50, 50, 3), dtype=np.uint8)
    z = O.cnn_logits(g, arch, w)
    x = O.normalize_input(g, arch.chan_mean)[..., 1]                   # channel 1
    x = np.maximum(x, 0)
    p1 = x.reshape(4, 25, 2, 25, 2).max(axis=(2, 4))
    p2 = p1[:, :24, :24].reshape(4, 12, 2, 12, 2).max(axis=(2, 4))
    assert np.array_equal(z, p2[:, 3, 5].astype(np.float32))


def _torch_forward(small, arch, w):
    """Independent forward with torch fp64 library ops on bf16-rounded tensors."""
    bf = lambda t: t.to(torch.float32).to(torch.bfloat16).to(torch.float64) if t.dtype != torch.float64 else \
        torch.from_numpy(O.bf16_round(t.numpy()))
    tobits = lambda b: torch.from_numpy(sg.bf16_bits_to_f32(b).astype(np.float64))
    g = torch.from_numpy(small.astype(np.float32))
    mu = torch.tensor(arch.chan_mean, dtype=torch.float32)
    x = torch.clamp((g - mu) / 127.5, -1.0, 1.0).to(torch.bfloat16).to(torch.float64)
    x = x.permute(0, 3, 1, 2)                                          # NCHW
    for l in range(arch.n_conv):
        wt = tobits(w["conv_w"][l]).permute(0, 3, 1, 2)                 # [Cout, Cin, 3, 3]
        b = torch.from_numpy(w["conv_b"][l].astype(np.float64))
        a = torch.nn.functional.conv2d(x, wt, b, padding=1)
        a = torch.nn.functional.max_pool2d(torch.relu(a), 2)           # floor mode
        x = bf(a)
    f = x.permute(0, 2, 3, 1).reshape(x.shape[0], -1)                  # (h, w, c)
    h1 = torch.relu(torch.nn.functional.linear(f, tobits(w["fc1_w"]),
                                               torch.from_numpy(w["fc1_b"].astype(np.float64))))
    h1 = bf(h1)
    z = h1 @ tobits(w["fc2_w"]) + float(w["fc2_b"][0])
    return z.to(torch.float32).numpy()


@pytest.mark.parametrize("arch", sg.ARCH_GRID + [sg.CnnArch(2, 16, 32), sg.CnnArch(4, 16, 256),
                                                 sg.CnnArch(2, 16, 64)], ids=lambda a: a.name)
def test_oracle_vs_torch_fp64(arch):
    w = sg.he_normal_weights(arch, 5)
    sc = sg.make_scene(sg.SceneSpec(50, 50, 60, seed=9, prevalence=0.5))
    small = sg.render_frames(sc, 0, 6)[:, :7500].reshape(6, 50, 50, 3)
    z = O.cnn_logits(small, arch, w)
    zt = _torch_forward(small, arch, w)
    # same bf16 rounding points, fp64 accumulation in a different order:
    # identical except where an fp64 reordering flips a bf16 tie (never seen)
    assert np.allclose(z, zt, atol=1e-6, rtol=0)
    assert np.std(z) > 0      # random weights give non-degenerate logits
