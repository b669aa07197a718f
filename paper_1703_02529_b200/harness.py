"""Evaluation harness: factor analysis and lesion study
 on the GPU cascade.

Host sequencing only: each row switches stages off in the configuration (reading
R-24: no skipping -> t_skip 1; no difference detector -> delta = -inf,
every checked frame fires; no specialized model -> (c_low, c_high) = (-inf, +inf),
every fired frame goes to the reference NN), runs noscope_cascade_run, scores the
labels with noscope_eval_labels (30-frame windows, 28 must agree),
and computes the modeled speedup N*T_full / (checked*T_mse [DD on] + fired*T_snn
[CNN on] + reference-NN frames*T_full) from the run's integer counts.
"""
from __future__ import annotations

import dataclasses
import math

from . import noscope as N

FACTOR_ROWS = [("oracle only", ()), ("+skipping", ("skip",)), ("+difference detection", ("skip", "dd")),
               ("+specialized model", ("skip", "dd", "cnn"))]
LESION_ROWS = [("full", ("skip", "dd", "cnn")), ("-skipping", ("dd", "cnn")),
               ("-difference detection", ("skip", "cnn")), ("-specialized model", ("skip", "dd"))]


def stage_config(dd: N.DD, lo: float, hi: float, stages):
    d = dataclasses.replace(dd, t_skip_frames=dd.t_skip_frames if "skip" in stages else 1,
                            delta_diff=dd.delta_diff if "dd" in stages else -math.inf)
    return d, (lo if "cnn" in stages else -math.inf), (hi if "cnn" in stages else math.inf)


def modeled_speedup(c: dict, stages, t_mse: int, t_snn: int, t_full: int) -> float:
    ref_frames = c["uncertain"] if "cnn" in stages else c["fired"]
    t = (c["checked"] * t_mse if "dd" in stages else 0) + (c["fired"] * t_snn if "cnn" in stages else 0) \
        + ref_frames * t_full
    return c["n"] * t_full / t


def factor_analysis(frames, width, height, dd: N.DD, arch: N.Arch, weights: N.Weights, lo, hi, labeller,
                    labeller_user, truth_dev, timing, rows=FACTOR_ROWS, window=30, agree_min=28):
    """frames: device u8 [n, pitch] (one unit); truth_dev: device u8 [n] reference labels."""
    out = []
    for name, stages in rows:
        d, l, h = stage_config(dd, lo, hi, stages)
        state = N.noscope_stream_state_init(d)
        res = N.noscope_cascade_run(d, arch, weights, l, h, frames, width, height, state, labeller,
                                    labeller_user, want_stats=True)
        st = res["stats"]
        cnt = dict(n=st["n_frames"], checked=st["n_frames"] - st["n_skipped"], fired=st["n_fired"],
                   uncertain=st["n_uncertain"])
        ev = N.noscope_eval_labels(res["labels"], truth_dev, window, agree_min)
        out.append(dict(name=name, accuracy=ev["correct_windows"] / ev["windows"], fp=ev["fp"], fn=ev["fn"],
                        speedup=modeled_speedup(cnt, stages, *timing), **cnt))
    return out
