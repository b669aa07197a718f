"""Pins of the oracle against the hand-derived values in tests/golden/oracle_pins.json.

These cover the rules that closed forms and invariants alone leave open (each was
shown unpinned by a mutation of the oracle in the round-1 review):
  * O1 box bounds at non-integer ratios (480 -> 50, 640 -> 50, 10 -> 4)
  * blocked-MSE remainder in the last block row / column
  * O4 order: the t_skip test comes before the mode-1 forced fire (R-8)
  * O8 labels of fired frames: NEG -> 0, POS -> 1, uncertain -> reference
Each fixture entry carries its citation and arithmetic."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_pins.json")))
DISP = {"K": O.SKIPPED, "S": O.SUPPRESSED, "F": O.FIRED}
ROUTE = {"NEG": O.R_NEG, "POS": O.R_POS, "UNC": O.R_UNC}


def _f(v):
    return {"+inf": math.inf, "-inf": -math.inf}.get(v, v) if isinstance(v, str) else float(v)


# ---------------- O1 ----------------
def _bright_row_frame(r=None, c=None):
    g = GOLD["downsample_box_bounds"]
    H, W = g["source_hw"]
    f = np.zeros((1, H, W, 3), np.uint8)
    if r is not None:
        f[0, r, :, :] = 255
    if c is not None:
        f[0, :, c, :] = 255
    return f


@pytest.mark.parametrize("case", GOLD["downsample_box_bounds"]["bright_row_cases"], ids=lambda c: f"row{c['row']}")
def test_downsample_row_bounds_480_to_50(case):
    g = O.downsample(_bright_row_frame(r=case["row"]), 50, 50)[0]
    lit = sorted(set(np.flatnonzero(g[:, :, 0].any(axis=1))))
    assert lit == [case["cell"]]
    assert np.all(g[case["cell"]] == case["value"])


@pytest.mark.parametrize("case", GOLD["downsample_box_bounds"]["bright_col_cases"], ids=lambda c: f"col{c['col']}")
def test_downsample_col_bounds_640_to_50(case):
    g = O.downsample(_bright_row_frame(c=case["col"]), 50, 50)[0]
    lit = sorted(set(np.flatnonzero(g[:, :, 0].any(axis=0))))
    assert lit == [case["cell"]]
    assert np.all(g[:, case["cell"]] == case["value"])


def test_downsample_cell_starts_480x640():
    g = GOLD["downsample_box_bounds"]
    # a lone bright row at each listed start lands in that cell; the row before it in the previous one
    for i, r0 in enumerate(g["row_starts_first_11"]):
        cells = np.flatnonzero(O.downsample(_bright_row_frame(r=r0), 50, 50)[0, :, 0, 0])
        assert list(cells) == [i]
        if r0 > 0:
            cells = np.flatnonzero(O.downsample(_bright_row_frame(r=r0 - 1), 50, 50)[0, :, 0, 0])
            assert list(cells) == [i - 1]
    for j, c0 in enumerate(g["col_starts_first_11"]):
        cells = np.flatnonzero(O.downsample(_bright_row_frame(c=c0), 50, 50)[0, 0, :, 0])
        assert list(cells) == [j]
        if c0 > 0:
            cells = np.flatnonzero(O.downsample(_bright_row_frame(c=c0 - 1), 50, 50)[0, 0, :, 0])
            assert list(cells) == [j - 1]


def test_downsample_ratio_2_5():
    g = GOLD["downsample_box_bounds"]["small_ratio_case"]
    f = np.zeros((1, 10, 3, 3), np.uint8)
    f[0, :, :, :] = np.asarray(g["source_rows"], np.uint8)[:, None, None]
    out = O.downsample(f, 4, 1)[0, :, 0, 0]
    assert list(out) == g["expected"]


# ---------------- O3 blocked remainder ----------------
@pytest.mark.parametrize("case", GOLD["blocked_mse_remainder"]["cases"],
                         ids=lambda c: f"{c['perturb']}{c['index']}")
def test_blocked_mse_remainder_in_last_block(case):
    g = GOLD["blocked_mse_remainder"]
    h, w = g["hw"]
    a = np.full((h, w, 3), 100, np.uint8)
    b = a.copy()
    if case["perturb"] == "row":
        b[case["index"], :, :] += case["delta"]
    else:
        b[:, case["index"], :] += case["delta"]
    assert list(O.blocked_mse(b, a, g["grid"])) == case["expected"]
    bounds = [list(x) for x in O.block_bounds(h, g["grid"])]
    assert bounds == g["row_bounds"]
    assert [list(x) for x in O.block_bounds(w, g["grid"])] == g["col_bounds"]


# ---------------- O4 order ----------------
@pytest.mark.parametrize("case", GOLD["skip_before_forced_fire"]["cases"], ids=lambda c: f"k{c['k']}s{c['t_skip']}")
def test_skip_before_forced_fire(case):
    n = case["n"]
    small = np.repeat(np.random.default_rng(5).integers(0, 256, (1, 50, 50, 3), dtype=np.uint8), n, axis=0)
    cfg = O.DDConfig(mode=case["mode"], metric=0, t_diff_frames=case["k"], t_skip_frames=case["t_skip"],
                     delta_diff=case["delta"])
    s, d = O.diff_detect(small, cfg)
    assert list(d) == [DISP[x] for x in case["disp"]]
    assert list(s) == [_f(x) for x in case["score"]]


# ---------------- O8 fired labels ----------------
def test_fired_frames_take_cnn_decision():
    g = GOLD["fired_labels"]
    disp = np.array([DISP[x] for x in g["disp"]], np.uint8)
    route = np.array([ROUTE[x] for x in g["route"]], np.uint8)
    L = O.resolve_labels(disp, route, np.array(g["labeller"], np.uint8), 0, 1, 1)
    assert list(L) == g["expected"]


def test_fired_labels_through_cascade_routing():
    # the same rule through route(): logits far below lo -> 0, far above hi -> 1, inside -> labeller
    z = np.float32([-5.0, 5.0, 0.0, 0.0])
    r = O.route(z, -1.0, 1.0)
    L = O.resolve_labels(np.full(4, O.FIRED, np.uint8), r, np.array([1, 0, 1, 0], np.uint8), 0, 1, 1)
    assert list(L) == [0, 1, 1, 0]


# ---------------- SPEC worked examples ----------------
@pytest.mark.parametrize("case", GOLD["spec_examples"]["mse"], ids=lambda c: c["cite"])
def test_spec_mse_examples(case):
    assert O.mse(np.array(case["a"]), np.array(case["b"])) == case["expected"]


def test_spec_quadrant_example():
    q = GOLD["spec_examples"]["quadrant"]
    a = np.full((*q["hw"], 3), q["base"], np.uint8)
    b = a.copy()
    (r0, r1), (c0, c1) = q["quadrant_rows"], q["quadrant_cols"]
    b[r0:r1, c0:c1] += q["delta"]
    assert list(O.blocked_mse(a, b, q["grid"])) == q["expected"]


# ---------------- O8 suppressed / skipped labels ----------------
@pytest.mark.parametrize("case", GOLD["mode1_suppressed_labels"]["cases"], ids=lambda c: f"mode{c['mode']}k{c['k']}")
def test_suppressed_labels_follow_anchor(case):
    disp = np.array([DISP[x] for x in case["disp"]], np.uint8)
    route = np.array([ROUTE.get(x, O.R_SUPP) for x in case["route"]], np.uint8)
    L = O.resolve_labels(disp, route, np.array(case["labeller"], np.uint8), case["mode"], case["k"], case["t_skip"])
    assert list(L) == case["expected"]


# ---------------- O6 input normalisation ----------------
@pytest.mark.parametrize("case", GOLD["normalize_clamp"]["cases"], ids=lambda c: f"G{c['G']}")
def test_normalize_clamp_and_bf16(case):
    x = O.normalize_input(np.full((1, 1, 1, 3), case["G"], np.uint8), (case["mu"],) * 3)
    assert np.all(x == case["expected"])
