"""Random-init specialized-CNN weights (He-normal, bf16) — generator only.

Architecture family (§4, Table 2, SURVEY.md
R-11/R-12): L conv layers of 3x3 'same' conv + ReLU + 2x2 maxpool with
filter doubling C*2^(l-1), then FC(D)+ReLU, FC(1) -> logit.  Weights are
drawn here as INPUTS; no forward arithmetic lives in this module.

Layout of every tensor (the ABI's noscope_cnn_weights, include/noscope.h):
  conv_w[l]  bf16 bits uint16 [Cout][3][3][Cin]
  conv_b[l]  float32 [Cout]
  fc1_w      bf16 bits uint16 [D][K], K ordered (h, w, c) of the last pooled map
  fc1_b      float32 [D]
  fc2_w      bf16 bits uint16 [D]
  fc2_b      float32 [1]
"""
from __future__ import annotations

import dataclasses
import itertools

import numpy as np


@dataclasses.dataclass(frozen=True)
class CnnArch:
    n_conv: int
    base_filters: int
    dense: int
    in_w: int = 50
    in_h: int = 50
    chan_mean: tuple = (127.5, 127.5, 127.5)

    def conv_channels(self):
        """[(Cin, Cout)] per conv layer (filter doubling)."""
        chans = []
        cin = 3
        for l in range(self.n_conv):
            cout = self.base_filters * (2 ** l)
            chans.append((cin, cout))
            cin = cout
        return chans

    def spatial(self):
        """Input spatial size of each conv layer plus the final pooled size."""
        h, w = self.in_h, self.in_w
        sizes = [(h, w)]
        for _ in range(self.n_conv):
            h, w = h // 2, w // 2
            sizes.append((h, w))
        return sizes

    def flat_dim(self):
        h, w = self.spatial()[-1]
        return h * w * self.conv_channels()[-1][1]

    @property
    def name(self):
        return f"L{self.n_conv}C{self.base_filters}D{self.dense}"


# BASELINE.json configs[2]: 2/4 conv layers x 32/64 filters x 32/128 dense
ARCH_GRID = [CnnArch(L, C, D) for L, C, D in itertools.product((2, 4), (32, 64), (32, 128))]
# the paper's model-search grid ("24 distinct configurations";
# Table 2 P:1136-1140 picks C = 16 for two videos): 2 L x 3 C x 4 D
PAPER_GRID = [CnnArch(L, C, D) for L, C, D in itertools.product((2, 4), (16, 32, 64), (32, 64, 128, 256))]


def bf16_round_f32(x) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), round-to-nearest-even.

    Used only to quantise freshly drawn random weights (inputs)."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(bits) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def he_normal_weights(arch: CnnArch, seed: int) -> dict:
    """Draw the weight set; returns dict of numpy arrays in the ABI layout."""
    rng = np.random.Generator(np.random.PCG64([seed, 97, arch.n_conv, arch.base_filters, arch.dense]))
    out = {"conv_w": [], "conv_b": []}
    for cin, cout in arch.conv_channels():
        std = np.sqrt(2.0 / (9 * cin))
        w = rng.normal(0.0, std, size=(cout, 3, 3, cin)).astype(np.float32)
        out["conv_w"].append(bf16_round_f32(w))
        out["conv_b"].append((0.01 * rng.normal(size=cout)).astype(np.float32))
    K, D = arch.flat_dim(), arch.dense
    out["fc1_w"] = bf16_round_f32(rng.normal(0.0, np.sqrt(2.0 / K), size=(D, K)).astype(np.float32))
    out["fc1_b"] = (0.01 * rng.normal(size=D)).astype(np.float32)
    out["fc2_w"] = bf16_round_f32(rng.normal(0.0, np.sqrt(1.0 / D), size=D).astype(np.float32))
    out["fc2_b"] = np.array([0.01 * rng.normal()], dtype=np.float32)
    return out


def zero_weights(arch: CnnArch) -> dict:
    out = {"conv_w": [], "conv_b": []}
    for cin, cout in arch.conv_channels():
        out["conv_w"].append(np.zeros((cout, 3, 3, cin), np.uint16))
        out["conv_b"].append(np.zeros(cout, np.float32))
    K, D = arch.flat_dim(), arch.dense
    out["fc1_w"] = np.zeros((D, K), np.uint16)
    out["fc1_b"] = np.zeros(D, np.float32)
    out["fc2_w"] = np.zeros(D, np.uint16)
    out["fc2_b"] = np.zeros(1, np.float32)
    return out


