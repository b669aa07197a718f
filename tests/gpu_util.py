"""Shared helpers for the GPU parity tests (inputs via synthgen, expectations via oracle)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg

requires_gpu = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")


def ns():
    from paper_1703_02529_b200 import noscope
    noscope.lib()
    return noscope


def scene_frames(W, H, n, seed, prevalence=0.3, sigma=2, stream=0):
    sc = sg.make_scene(sg.SceneSpec(W, H, n, seed=seed, stream=stream, prevalence=prevalence,
                                    noise_sigma=sigma))
    fr = sg.render_frames(sc)
    return sc, fr


def hw3(fr, W, H):
    return fr[:, :W * H * 3].reshape(-1, H, W, 3)


def dd_pair(ns_mod, mode, metric, out=50, grid=10, k=5, t_skip=1, delta=20.0, ref=None, lr=None,
            device="cuda"):
    """Matching (oracle DDConfig, binding DD) pair."""
    lr_w, lr_b = lr if lr is not None else (None, 0.0)
    ocfg = O.DDConfig(mode=mode, metric=metric, out_w=out, out_h=out, grid=grid, t_diff_frames=k,
                      t_skip_frames=t_skip, delta_diff=delta, ref_image=ref, lr_w=lr_w, lr_b=lr_b)
    g = ns_mod.DD(mode=mode, metric=metric, out_w=out, out_h=out, grid=grid, t_diff_frames=k,
                  t_skip_frames=t_skip, delta_diff=delta,
                  ref_image=None if ref is None else torch.from_numpy(np.ascontiguousarray(ref)).to(device),
                  lr_weights=None if lr_w is None else torch.from_numpy(lr_w).to(device),
                  lr_bias=float(lr_b))
    return ocfg, g


def pick_thresholds_in_gaps(z, tol, lo_q=0.3, hi_q=0.7):
    """Choose lo < hi at midpoints of the widest gaps of sorted logits near the
    requested quantiles; returns (lo, hi, margin) where margin = distance from
    each threshold to the nearest logit."""
    zs = np.sort(np.asarray(z, np.float64))
    if len(zs) < 4:
        return -math.inf, math.inf, math.inf
    gaps = np.diff(zs)

    def best_gap(q):
        c = int(q * (len(zs) - 1))
        lo_i, hi_i = max(0, c - len(zs) // 6), min(len(gaps), c + len(zs) // 6 + 1)
        i = lo_i + int(np.argmax(gaps[lo_i:hi_i]))
        return 0.5 * (zs[i] + zs[i + 1]), 0.5 * gaps[i]

    lo, m1 = best_gap(lo_q)
    hi, m2 = best_gap(hi_q)
    if lo > hi:
        lo, hi = hi, lo
    return float(np.float32(lo)), float(np.float32(hi)), min(m1, m2)
