"""Mutation check of the oracle's pins: apply one plausible mistake at a time to a
temporary copy of oracle/ and require that the CPU suite (-m "not gpu") fails.

Each mutation is a rule the round-1 review showed unpinned, plus a few more
(dropped terms, swapped operands).  Usage: python tools/oracle_mutations.py
Prints one line per mutation: name, failing-test count, first failing test."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    # O1 box bounds: ceil instead of floor at non-integer ratios
    "O1_ceil_row_bounds": ("r0, r1 = (i * H) // out_h, ((i + 1) * H) // out_h",
                           "r0, r1 = -((-i * H) // out_h), -((-(i + 1) * H) // out_h)"),
    "O1_ceil_col_bounds": ("q0, q1 = (j * W) // out_w, ((j + 1) * W) // out_w",
                           "q0, q1 = -((-j * W) // out_w), -((-(j + 1) * W) // out_w)"),
    "O1_round_half_down": ("((2 * S + n) // (2 * n))", "((2 * S + n - 1) // (2 * n))"),
    # O8 fired labels swapped
    "O8_neg_pos_swapped": ("L[t] = 0 if r == R_NEG else 1 if r == R_POS else labeller[t]",
                           "L[t] = 1 if r == R_NEG else 0 if r == R_POS else labeller[t]"),
    # O4 forced fire before the t_skip test
    "O4_forced_fire_first": ("""        if tau % cfg.t_skip_frames != 0:
            score[tau], disp[tau] = -math.inf, SKIPPED
            continue
        if cfg.mode == 1 and tau < k:
            score[tau], disp[tau] = math.inf, FIRED
            continue
""", """        if cfg.mode == 1 and tau < k:
            score[tau], disp[tau] = math.inf, FIRED
            continue
        if tau % cfg.t_skip_frames != 0:
            score[tau], disp[tau] = -math.inf, SKIPPED
            continue
"""),
    "O4_non_strict_fire": ("disp[tau] = FIRED if s > cfg.delta_diff else SUPPRESSED",
                           "disp[tau] = FIRED if s >= cfg.delta_diff else SUPPRESSED"),
    # O3 remainder given to the first block instead of the last
    "O3_remainder_first_block": ("return [(k * step, (k + 1) * step if k < g - 1 else n) for k in range(g)]",
                                 "r = n - step * g\n    return [(0 if k == 0 else k * step + r, (k + 1) * step + r) for k in range(g)]"),
    "O3_logit_drops_bias": ("z = float(np.float32(bias))", "z = 0.0"),
    # (L[t] = L[t - 1] for skipped frames is an equivalent mutant: by induction the
    #  previous frame of a skip period already holds the period's checked label)
    "O8_skip_copies_first": ("L[t] = L[t - (t % t_skip)]", "L[t] = L[0]"),
    "O8_mode1_suppressed_zero": ("L[t] = 0 if mode == 0 else L[t - k]", "L[t] = 0"),
    # O7 equality routed as confident
    "O7_equal_lo_negative": ("if zi < lo32:", "if zi <= lo32:"),
    # O6 pool / normalisation
    "O6_no_clamp": ("x = np.minimum(np.maximum(x, np.float32(-1.0)), np.float32(1.0))", "x = x"),
    "O6_transposed_tap": ("acc += xp[:, dy:dy + H, dx:dx + W, :] @ w[:, dy, dx, :].T",
                          "acc += xp[:, dx:dx + H, dy:dy + W, :] @ w[:, dy, dx, :].T"),
    # O9 sweep
    "O9_GE_strict": ('T["GE"][j, t] = (fired & (z >= u[t])).sum()', 'T["GE"][j, t] = (fired & (z > u[t])).sum()'),
    "O9_cost_drops_snn": ("return checked * t_mse + F * t_snn + U * t_full", "return checked * t_mse + U * t_full"),
    # N4 training stop rule: validation instead of training loss
    "N4_stop_on_val_loss": ("if e > 0 and hist[e][0] > hist[e - 1][0]:", "if e > 0 and hist[e][1] > hist[e - 1][1]:"),
    # N1 LR fit: gradient without the l2 term
    "N1_lr_no_l2_grad": ("g = X1.T @ (p - t) / n + reg * v", "g = X1.T @ (p - t) / n"),
    "N1_lr_sign_error": ("delta = -np.linalg.solve(", "delta = np.linalg.solve("),
    "N1_lr_unscale_bias": ("return w / sd, v[d] - float(np.sum(w * mu / sd))", "return w / sd, v[d]"),
    "N1_ref_round_down": ("return ((2 * S + m) // (2 * m)).astype(np.uint8)", "return (S // m).astype(np.uint8)"),
    "N1_ref_uses_positives": ("neg = np.asarray(labels) == 0", "neg = np.asarray(labels) != 0"),
    "N1_features_wrong_anchor": ("out[i] = blocked_mse(small[i], small[i - k], grid)",
                                 "out[i] = blocked_mse(small[i], small[i - k + 1], grid)"),
    "N1_sample_std": ("sd = F.std(axis=0)\n    sd = np.where(sd > 0, sd, 1.0)\n    X = (F - mu) / sd",
                      "sd = F.std(axis=0, ddof=1)\n    sd = np.where(sd > 0, sd, 1.0)\n    X = (F - mu) / sd"),
    # O9 record builder and tables
    "O9_records_mode1_no_lag": ("a[i] = 0 if (mode == 0 or i < k) else y[i - k]", "a[i] = 0 if (mode == 0 or i < k) else y[i]"),
    "O9_records_skip_current": ("a[i] = y[last_checked]", "a[i] = y[i]"),
    "O9_FPnf_wrong_cell": ('T["FPnf"][j] = (nf & (a == 1) & (y == 0)).sum()', 'T["FPnf"][j] = (nf & (a == 0) & (y == 1)).sum()'),
    "O9_fired_non_strict": ("fired = s > delta[j]", "fired = s >= delta[j]"),
    "O9_tiebreak_min_low": ("key = (c, U, j, -l, h)", "key = (c, U, j, l, h)"),
    # N3 evaluation
    "N3_window_strict": ("return float((per >= agree_min).sum()) / nw", "return float((per > agree_min).sum()) / nw"),
    "N3_speedup_drops_snn": ('+ (c["fired"] * t_snn if "cnn" in stages else 0)', '+ 0'),
    # N4 training: best epoch on ties / by training loss
    "N4_best_by_train_loss": ("if val < best_val:", "if tot / len(perm) < best_val:"),
}


def run_one(name, old, new):
    d = tempfile.mkdtemp(prefix=f"mut_{name}_")
    try:
        for sub in ("oracle", "synthgen", "tests", "paper_1703_02529_b200", "include"):
            shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                            ignore=shutil.ignore_patterns("__pycache__", "*.so"))
        for f in ("pytest.ini", "bench.py"):
            shutil.copy(os.path.join(ROOT, f), d)
        p = os.path.join(d, "oracle", "noscope_oracle.py")
        s = open(p).read()
        if old not in s:
            return name, None, "mutation site not found"
        open(p, "w").write(s.replace(old, new, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-q", "-m", "not gpu and not slow",
                            "-p", "no:cacheprovider", "-k", "oracle or golden"],
                           cwd=d, capture_output=True, text=True, timeout=1800)
        failed = [l.split()[1] for l in r.stdout.splitlines() if l.startswith("FAILED")]
        return name, len(failed), failed[0] if failed else "-"
    finally:
        shutil.rmtree(d, ignore_errors=True)


def main():
    names = sys.argv[1:] or list(MUTATIONS)
    bad = 0
    for n in names:
        name, nfail, first = run_one(n, *MUTATIONS[n])
        ok = bool(nfail)
        bad += not ok
        print(f"{'caught ' if ok else 'MISSED '} {name:28s} failing={nfail} first={first}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
