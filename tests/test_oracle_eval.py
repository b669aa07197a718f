"""Pins of the oracle's evaluation harness: SPEC's worked
examples for windowed accuracy, FP/FN and modeled speedup,
and the factor-analysis / lesion invariants."""
import math

import numpy as np
import pytest

import oracle as O
import synthgen as sg


def test_windowed_accuracy_examples():
    r = np.zeros(90, np.uint8)
    assert O.windowed_accuracy(r, r) == 1.0                              # pred == ref
    p = r.copy()
    p[:2] = 1
    assert O.windowed_accuracy(p[:30], r[:30]) == 1.0                   # 28/30 agree -> correct
    p[2] = 1
    assert O.windowed_accuracy(p[:30], r[:30]) == 0.0                   # 27/30 -> incorrect
    q = r.copy()
    q[30:32] = 1                    # window 2: 28/30
    q[60:70] = 1                    # window 3: 20/30
    assert O.windowed_accuracy(q, r) == pytest.approx(2 / 3)
    assert O.windowed_accuracy(np.zeros(95), np.zeros(95)) == 1.0       # partial window dropped
    with pytest.raises(ValueError):
        O.windowed_accuracy(np.zeros(30), np.zeros(31))


def test_fp_fn_examples():
    assert O.fp_fn([1, 0, 0, 1], [1, 1, 0, 0])[:2] == (1, 1)
    fp, fn, tp, tn = O.fp_fn(np.ones(10), np.zeros(10))
    assert (fp, fn, tp, tn) == (10, 0, 0, 0)
    assert sum(O.fp_fn(np.arange(7) % 2, np.arange(7) % 3 == 0)) == 7


def test_modeled_speedup_closed_forms():
    c = dict(n=100, checked=100, fired=100, uncertain=100)
    assert O.modeled_speedup(c, (), 1, 10, 1000) == 1.0                 # all to oracle
    c = dict(n=150, checked=10, fired=4, uncertain=1)
    assert O.modeled_speedup(c, ("skip", "dd", "cnn"), 2, 30, 1000) == 150 * 1000 / (20 + 120 + 1000)
    assert O.modeled_speedup(c, ("skip", "dd"), 2, 30, 1000) == 150 * 1000 / (20 + 4000)


def _clip():
    n, W = 90, 40
    sc = sg.make_scene(sg.SceneSpec(W, W, n, seed=13, prevalence=0.4, noise_sigma=2))
    fr = sg.render_frames(sc)[:, :W * W * 3].reshape(n, W, W, 3)
    cfg = O.DDConfig(mode=0, metric=0, out_w=W, out_h=W, t_skip_frames=3, delta_diff=15.0,
                     ref_image=sg.background(sc.spec))
    return fr, cfg, sc.truth[:n].astype(np.uint8)


def test_factor_analysis_invariants(monkeypatch):
    fr, cfg, y = _clip()
    # a stand-in "specialized model": logits from a fixed function of the frame
    monkeypatch.setattr(O.noscope_oracle, "cnn_logits",
                        lambda sm, arch, w: (sm.reshape(len(sm), -1).astype(np.float64).mean(1) - 60.0)
                        .astype(np.float32))
    rows = O.factor_analysis(fr, cfg, None, None, -1.0, 1.0, y, (2, 30, 1000))
    assert rows[0]["accuracy"] == 1.0 and rows[0]["speedup"] == 1.0
    assert rows[0]["fp"] == rows[0]["fn"] == 0
    assert rows[1]["checked"] == math.ceil(90 / 3)                      # ceil(N/t_skip)
    assert rows[1]["speedup"] == pytest.approx(90 / 30)
    les = O.factor_analysis(fr, cfg, None, None, -1.0, 1.0, y, (2, 30, 1000), rows=O.LESION_ROWS)
    # ("removing a stage never increases speedup" is a property of SPEC's golden
    # clip, not an identity: a DD that suppresses little can cost more than it saves)
    no_dd = les[2]
    assert no_dd["fired"] == no_dd["checked"]                           # nothing suppressed
    no_cnn = les[3]
    assert no_cnn["uncertain"] == no_cnn["fired"]                       # fired -> oracle
    assert les[0]["name"] == "full" and les[0]["speedup"] == rows[3]["speedup"]
