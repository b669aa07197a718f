"""Plain, slow CPU oracle of NoScope's per-frame cascade and CBO threshold sweep.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It shares no
code with the CUDA path (paper_1703_02529_b200/) and never imports it.

Each function is the plain definition written out from PAPER.md (P:n = line n
of /root/reference/PAPER.md); where the paper is silent the reading adopted is
SURVEY.md §8(c) O1-O10 / R-1..R-20, listed again in DESIGN.md "Readings".
Arithmetic: integers are exact (Python/numpy int64); floating point is fp64
unless the definition fixes another precision (the fp32 normalisation O6 and
fp32 logit comparisons O7, the bf16 roundings of the CNN's activations).

Parity status per function: every function below is
pinned by tests/test_oracle_*.py against closed forms, library routines or
brute force, except cnn_logits on random weights, which is pinned by closed
forms on special weights plus an independent torch-fp64 re-derivation of the
layer algebra (tests/test_oracle_cnn.py).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# Disposition codes (O4; SPEC dd_step S:227-235)
SKIPPED, SUPPRESSED, FIRED = 0, 1, 2
# Per-frame route codes (ABI route_out): 0 skip, 1 suppressed, 2 neg, 3 pos, 4 uncertain
R_SKIP, R_SUPP, R_NEG, R_POS, R_UNC = 0, 1, 2, 3, 4


# --------------------------------------------------------------------------
# O1 Downsample — P:834-837 "resizes them for downstream processing";
#    area averaging S:74; reading R-1 (integer box filter, round half up)
# --------------------------------------------------------------------------
def downsample(frames: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    """frames uint8 [N, H, W, 3] -> uint8 [N, out_h, out_w, 3].

    G[i][j][c] = floor((2*S + n) / (2*n)), S = sum of F over rows
    [floor(iH/h), floor((i+1)H/h)) x cols [floor(jW/w), floor((j+1)W/w)),
    n = #rows * #cols.  h > H or w > W is an error."""
    N, H, W, C = frames.shape
    if out_h > H or out_w > W:
        raise ValueError("downsample target larger than source (S:75)")
    out = np.empty((N, out_h, out_w, C), dtype=np.uint8)
    f = frames.astype(np.int64)
    for i in range(out_h):
        r0, r1 = (i * H) // out_h, ((i + 1) * H) // out_h
        for j in range(out_w):
            q0, q1 = (j * W) // out_w, ((j + 1) * W) // out_w
            n = (r1 - r0) * (q1 - q0)
            S = f[:, r0:r1, q0:q1, :].sum(axis=(1, 2))          # [N, C] exact
            out[:, i, j, :] = ((2 * S + n) // (2 * n)).astype(np.uint8)
    return out


# --------------------------------------------------------------------------
# O3 Scores — P:575-585 "computes the Mean Square Error (MSE) between them";
#    blocked: "subdivides each image into a grid and computes the metric on
#    every grid block ... trains a logistic regression (LR) classifier to weigh
#    each block"; readings R-2 (raw u8, all channels), R-3 (logit, no sigmoid)
# --------------------------------------------------------------------------
def ssd(a: np.ndarray, b: np.ndarray) -> int:
    """Exact sum of squared differences over all elements (integer)."""
    d = a.astype(np.int64) - b.astype(np.int64)
    return int((d * d).sum())


def mse(a: np.ndarray, b: np.ndarray) -> float:
    """MSE = (double)SSD / (double)count (correctly rounded ratio)."""
    return float(ssd(a, b)) / float(a.size)


def block_bounds(n: int, g: int):
    """Block k covers [k*floor(n/g), (k+1)*floor(n/g)); the last takes the
    remainder."""
    step = n // g
    return [(k * step, (k + 1) * step if k < g - 1 else n) for k in range(g)]


def blocked_mse(a: np.ndarray, b: np.ndarray, g: int) -> np.ndarray:
    """a, b: [h, w, 3].  Returns float64 [g*g] block MSEs in row-major block order."""
    h, w = a.shape[0], a.shape[1]
    out = np.empty(g * g, dtype=np.float64)
    for bi, (r0, r1) in enumerate(block_bounds(h, g)):
        for bj, (c0, c1) in enumerate(block_bounds(w, g)):
            blk_a, blk_b = a[r0:r1, c0:c1], b[r0:r1, c0:c1]
            out[bi * g + bj] = float(ssd(blk_a, blk_b)) / float(blk_a.size)
    return out


def lr_logit(m: np.ndarray, w: np.ndarray, bias) -> float:
    """z = b; z = z + w_k*m_k for k in order, each product and sum rounded
    to fp64 separately (plain Python floats: no fused multiply-add)."""
    z = float(np.float32(bias))
    for k in range(len(m)):
        z = z + float(np.float32(w[k])) * float(m[k])
    return z


def score_frame(G: np.ndarray, A: np.ndarray, metric: int, grid: int = 1,
                lr_w=None, lr_b=0.0) -> float:
    if metric == 0:
        return mse(G, A)
    return lr_logit(blocked_mse(G, A, grid), lr_w, lr_b)


# --------------------------------------------------------------------------
# O2/O4 Difference detector over one unit — P:554-563 (reference image / an
#   earlier frame t_diff back), P:587-593 and P:678-679 ("fire if the frame's
#   MSE ... is higher than delta_diff"), P:601-610 (check every t_skip frames);
#   readings R-4 (strict >), R-8 (fixed lag k, tau<k forced fire), R-10.
# --------------------------------------------------------------------------
@dataclasses.dataclass
class DDConfig:
    mode: int = 0            # 0 reference image, 1 earlier frame t-k
    metric: int = 0          # 0 global MSE, 1 blocked MSE + LR
    out_w: int = 50
    out_h: int = 50
    grid: int = 1
    t_diff_frames: int = 1   # k
    t_skip_frames: int = 1
    delta_diff: float = 0.0
    ref_image: np.ndarray | None = None    # uint8 [out_h, out_w, 3]
    lr_w: np.ndarray | None = None         # float32 [grid*grid]
    lr_b: float = 0.0


def diff_detect(small: np.ndarray, cfg: DDConfig):
    """small: uint8 [N, h, w, 3] downsampled frames of ONE unit (tau = 0..N-1).

    Returns (score float64[N], disposition uint8[N]).  Skipped frames carry
    score -inf, forced fires (mode 1, tau < k) +inf."""
    N = small.shape[0]
    score = np.empty(N, dtype=np.float64)
    disp = np.empty(N, dtype=np.uint8)
    k = cfg.t_diff_frames
    for tau in range(N):
        if tau % cfg.t_skip_frames != 0:
            score[tau], disp[tau] = -math.inf, SKIPPED
            continue
        if cfg.mode == 1 and tau < k:
            score[tau], disp[tau] = math.inf, FIRED
            continue
        anchor = cfg.ref_image if cfg.mode == 0 else small[tau - k]
        s = score_frame(small[tau], anchor, cfg.metric, cfg.grid, cfg.lr_w, cfg.lr_b)
        score[tau] = s
        disp[tau] = FIRED if s > cfg.delta_diff else SUPPRESSED
    return score, disp


# --------------------------------------------------------------------------
# O5 Compaction — batches for the specialized NN
# --------------------------------------------------------------------------
def compact(disp: np.ndarray) -> np.ndarray:
    """Ascending int32 indices t with disp[t] == FIRED."""
    return np.array([t for t in range(len(disp)) if disp[t] == FIRED], dtype=np.int32)


# --------------------------------------------------------------------------
# O6 Specialized CNN — P:437-456 ("AlexNet ... filter doubling ... ReLU ...
#   softmax"), P:449-453 (layers 2/4, filters 32/64, dense 32..256),
#   P:866-869 (mean-centre, range [-1, 1]); readings R-11, R-12, R-13.
# --------------------------------------------------------------------------
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 (8 significant bits), ties to
    even, returned as float64.  Normal range only (activations never reach
    bf16 subnormals or overflow)."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                      # x = m * 2^e, |m| in [0.5, 1)
    return np.ldexp(np.rint(m * 256.0), e - 8)


def normalize_input(G: np.ndarray, chan_mean) -> np.ndarray:
    """x = bf16_RNE(clamp(((float)G - mu_c) / 127.5f, -1, 1)) in fp32 IEEE."""
    g = G.astype(np.float32)
    mu = np.asarray(chan_mean, dtype=np.float32)
    x = (g - mu) / np.float32(127.5)
    x = np.minimum(np.maximum(x, np.float32(-1.0)), np.float32(1.0))
    return bf16_round(x.astype(np.float64))


def bf16_bits_to_f64(bits) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def conv3x3_same(x: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """x [n, H, W, Cin] f64, w [Cout, 3, 3, Cin] f64, b [Cout] -> [n, H, W, Cout]
    acc = b + sum_{dy,dx,ci} w[co,dy,dx,ci] * x[y+dy-1, x+dx-1, ci] (zero pad 1),
    accumulated in fp64 (a library matmul per tap)."""
    n, H, W, _ = x.shape
    xp = np.zeros((n, H + 2, W + 2, x.shape[3]), dtype=np.float64)
    xp[:, 1:H + 1, 1:W + 1, :] = x
    acc = np.broadcast_to(b.astype(np.float64), (n, H, W, w.shape[0])).copy()
    for dy in range(3):
        for dx in range(3):
            acc += xp[:, dy:dy + H, dx:dx + W, :] @ w[:, dy, dx, :].T
    return acc


def maxpool2x2_floor(x: np.ndarray) -> np.ndarray:
    """2x2 stride-2 max pool, floor (50->25->12->6->3)."""
    n, H, W, C = x.shape
    Ho, Wo = H // 2, W // 2
    v = x[:, :2 * Ho, :2 * Wo, :].reshape(n, Ho, 2, Wo, 2, C)
    return v.max(axis=(2, 4))


def cnn_logits(small: np.ndarray, arch, weights: dict, batch: int = 256) -> np.ndarray:
    """small uint8 [n, in_h, in_w, 3] -> fp32 logits z [n].

    Per layer l: 3x3 same conv (fp64 acc + bias) -> ReLU -> 2x2 maxpool ->
    round to bf16.  Flatten (h, w, c) -> FC1 (fp64 acc + bias) -> ReLU ->
    bf16 -> FC2 (fp64 acc) + b2 -> z = (float)z.  c = sigmoid(z) is the
    paper's confidence (2-class softmax == sigmoid of the logit gap)."""
    n = small.shape[0]
    out = np.empty(n, dtype=np.float32)
    conv_w = [bf16_bits_to_f64(w) for w in weights["conv_w"]]
    conv_b = [np.asarray(b, dtype=np.float32).astype(np.float64) for b in weights["conv_b"]]
    fc1_w = bf16_bits_to_f64(weights["fc1_w"])
    fc1_b = np.asarray(weights["fc1_b"], dtype=np.float32).astype(np.float64)
    fc2_w = bf16_bits_to_f64(weights["fc2_w"])
    fc2_b = float(np.asarray(weights["fc2_b"], dtype=np.float32)[0])
    for s in range(0, n, batch):
        x = normalize_input(small[s:s + batch], arch.chan_mean)
        for l in range(arch.n_conv):
            a = conv3x3_same(x, conv_w[l], conv_b[l])
            a = np.maximum(a, 0.0)
            x = bf16_round(maxpool2x2_floor(a))
        f = x.reshape(x.shape[0], -1)                          # (h, w, c) order
        h1 = bf16_round(np.maximum(f @ fc1_w.T + fc1_b, 0.0))
        z = h1 @ fc2_w + fc2_b
        out[s:s + batch] = z.astype(np.float32)
    return out


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-np.asarray(z, dtype=np.float64)))


# --------------------------------------------------------------------------
# O7 Routing — P:377-380 / P:458-462: "no object" if c < c_low, "object" if
#   c > c_high, else call the reference NN; reading R-5 (strict confident
#   decisions, equality -> uncertain, compared on fp32 logits).
# --------------------------------------------------------------------------
def route(z: np.ndarray, lo: float, hi: float) -> np.ndarray:
    if not lo <= hi:
        raise ValueError("c_low must not exceed c_high (S:280)")
    out = np.empty(len(z), dtype=np.uint8)
    lo32, hi32 = np.float32(lo), np.float32(hi)
    for i, zi in enumerate(np.asarray(z, dtype=np.float32)):
        if zi < lo32:
            out[i] = R_NEG
        elif zi > hi32:
            out[i] = R_POS
        else:
            out[i] = R_UNC
    return out


# --------------------------------------------------------------------------
# O8 Labels — P:559-563 ("returns the same labels that it output for the
#   previous frame"), P:554-558 (reference image contains no objects),
#   P:601-610 (skipped frames); readings R-9, R-10.
# --------------------------------------------------------------------------
def resolve_labels(disp: np.ndarray, fired_route: np.ndarray, labeller: np.ndarray,
                   mode: int, k: int, t_skip: int) -> np.ndarray:
    """disp uint8[N]; fired_route uint8[N] (route code for fired frames, else
    ignored); labeller uint8[N] (reference answer, read only for uncertain
    frames).  One forward loop; every pointer is strictly backward."""
    N = len(disp)
    L = np.zeros(N, dtype=np.uint8)
    for t in range(N):
        d = disp[t]
        if d == SKIPPED:
            L[t] = L[t - (t % t_skip)]
        elif d == SUPPRESSED:
            L[t] = 0 if mode == 0 else L[t - k]
        else:
            r = fired_route[t]
            L[t] = 0 if r == R_NEG else 1 if r == R_POS else labeller[t]
    return L


def cascade(frames_hw3: np.ndarray, cfg: DDConfig, arch, weights, lo: float, hi: float,
            truth: np.ndarray):
    """Whole per-unit cascade: downsample -> DD -> compaction ->
    CNN -> routing -> stand-in labeller (ground truth) -> labels.

    Returns dict with small, score, disp, idx, logits (fired only), route
    (per-frame code), labels."""
    small = downsample(frames_hw3, cfg.out_h, cfg.out_w)
    score, disp = diff_detect(small, cfg)
    idx = compact(disp)
    z = cnn_logits(small[idx], arch, weights) if len(idx) else np.zeros(0, np.float32)
    r_fired = route(z, lo, hi)
    route_pf = np.where(disp == SKIPPED, R_SKIP, R_SUPP).astype(np.uint8)
    route_pf[idx] = r_fired
    labels = resolve_labels(disp, route_pf, truth, cfg.mode, cfg.t_diff_frames,
                            cfg.t_skip_frames)
    return dict(small=small, score=score, disp=disp, idx=idx, logits=z,
                route=route_pf, labels=labels)


# --------------------------------------------------------------------------
# O9 CBO threshold sweep — P:627-637 (objective), P:685-701 (cost model,
#   formula P:696), P:747-779 (sort by delta, sweep prefixes, move c_low up /
#   c_high down until FN*/FP*); readings R-6, R-7, R-14, R-15, R-16, R-17.
# --------------------------------------------------------------------------
def build_records(score: np.ndarray, y: np.ndarray, mode: int, k: int):
    """Default record builder (S:439 approximation): a_i = label the cascade
    would inherit if frame i is not fired, computed from reference labels y:
    skipped -> y[last checked]; mode 0 -> 0; mode 1 -> y[i-k] (0 if i<k)."""
    N = len(score)
    a = np.zeros(N, dtype=np.uint8)
    last_checked = 0
    for i in range(N):
        if score[i] == -math.inf:
            a[i] = y[last_checked]
        else:
            last_checked = i
            a[i] = 0 if (mode == 0 or i < k) else y[i - k]
    return a


def sweep_tables(s, z, y, a, delta, u):
    """Direct per-threshold counts (O9).  Returns dict of uint64 tables:
    F[j], FPnf[j], FNnf[j], FPf[j][h], FNf[j][l], GE[j][l] = #(fired, z >= u_l),
    GT[j][h] = #(fired, z > u_h), plus checked and total counts."""
    s = np.asarray(s, np.float64); z = np.asarray(z, np.float32)
    y = np.asarray(y, np.uint8); a = np.asarray(a, np.uint8)
    nd, m = len(delta), len(u)
    T = {k: np.zeros((nd, m), np.uint64) for k in ("FPf", "FNf", "GE", "GT")}
    for k in ("F", "FPnf", "FNnf"):
        T[k] = np.zeros(nd, np.uint64)
    for j in range(nd):
        fired = s > delta[j]
        nf = ~fired
        T["F"][j] = fired.sum()
        T["FPnf"][j] = (nf & (a == 1) & (y == 0)).sum()
        T["FNnf"][j] = (nf & (a == 0) & (y == 1)).sum()
        for t in range(m):
            T["FPf"][j, t] = (fired & (z > u[t]) & (y == 0)).sum()
            T["FNf"][j, t] = (fired & (z < u[t]) & (y == 1)).sum()
            T["GE"][j, t] = (fired & (z >= u[t])).sum()
            T["GT"][j, t] = (fired & (z > u[t])).sum()
    T["checked"] = int((s != -math.inf).sum())
    T["total"] = len(s)
    return T


def triple_counts(T, j, l, h):
    """FP, FN, F, U of triple (delta_j, u_l, u_h), l <= h."""
    fp = int(T["FPnf"][j]) + int(T["FPf"][j, h])
    fn = int(T["FNnf"][j]) + int(T["FNf"][j, l])
    U = int(T["GE"][j, l]) - int(T["GT"][j, h])     # #(fired, u_l <= z <= u_h)
    return fp, fn, int(T["F"][j]), U


def cost_ps(checked, F, U, t_mse, t_snn, t_full):
    """N x (f_s T_MSE + f_s f_m T_SNN + f_s f_m f_c T_Full) in integer
    picoseconds: f_s = checked/N, f_s f_m = F/N, f_s f_m f_c = U/N."""
    return checked * t_mse + F * t_snn + U * t_full


def sweep_best(T, timing, fp_limit, fn_limit):
    """argmin over feasible (j, l <= h) of the key (cost, U, j, -l, h); if none
    is feasible, the best-effort triple minimising (max violation, cost, U, j,
    -l, h) with feasible=False (R-14)."""
    nd, m = T["FPf"].shape
    best, best_key = None, None
    fb, fb_key = None, None
    for j in range(nd):
        for l in range(m):
            for h in range(l, m):
                fp, fn, F, U = triple_counts(T, j, l, h)
                c = cost_ps(T["checked"], F, U, *timing)
                rec = dict(j=j, l=l, h=h, fp=fp, fn=fn, F=F, U=U, cost=c)
                if fp <= fp_limit and fn <= fn_limit:
                    key = (c, U, j, -l, h)
                    if best_key is None or key < best_key:
                        best, best_key = rec, key
                else:
                    viol = max(fp - fp_limit, fn - fn_limit, 0)
                    key = (viol, c, U, j, -l, h)
                    if fb_key is None or key < fb_key:
                        fb, fb_key = rec, key
    if best is not None:
        best["feasible"] = True
        return best
    fb["feasible"] = False
    return fb


def sweep(s, z, y, a, delta, u, timing, fp_limit, fn_limit):
    T = sweep_tables(s, z, y, a, delta, u)
    return T, sweep_best(T, timing, fp_limit, fn_limit)


def sweep_brute_force(s, z, y, a, delta, u, timing, fp_limit, fn_limit):
    """Pure-Python brute force over ALL triples and ALL records (tiny inputs):
    simulate the cascade per triple and count errors directly."""
    t_mse, t_snn, t_full = timing
    checked = sum(1 for v in s if v != -math.inf)
    best, best_key, fb, fb_key = None, None, None, None
    for j in range(len(delta)):
        for l in range(len(u)):
            for h in range(l, len(u)):
                fp = fn = F = U = 0
                for i in range(len(s)):
                    if s[i] > delta[j]:
                        F += 1
                        zi = np.float32(z[i])
                        if zi < u[l]:
                            out = 0
                        elif zi > u[h]:
                            out = 1
                        else:
                            out = int(y[i]); U += 1
                    else:
                        out = int(a[i])
                    fp += int(out == 1 and y[i] == 0)
                    fn += int(out == 0 and y[i] == 1)
                c = checked * t_mse + F * t_snn + U * t_full
                rec = dict(j=j, l=l, h=h, fp=fp, fn=fn, F=F, U=U, cost=c)
                if fp <= fp_limit and fn <= fn_limit:
                    key = (c, U, j, -l, h)
                    if best_key is None or key < best_key:
                        best, best_key = rec, key
                else:
                    key = (max(fp - fp_limit, fn - fn_limit, 0), c, U, j, -l, h)
                    if fb_key is None or key < fb_key:
                        fb, fb_key = rec, key
    if best is not None:
        best["feasible"] = True
        return best
    fb["feasible"] = False
    return fb


def sweep_greedy_paper(s, z, y, a, delta, u, timing, fp_limit, fn_limit):
    """The paper's own procedure: for each delta prefix, start with
    thresholds at the extremes, move c_low up while FN stays within FN*, move
    c_high down while FP stays within FP*; if they cross, meet at the candidate
    in [h_min, l_max] minimising U (R-15).  Used as an equivalence pin."""
    t_mse, t_snn, t_full = timing
    T = sweep_tables(s, z, y, a, delta, u)
    m = len(u)
    cands = []
    for j in range(len(delta)):
        if T["FPnf"][j] + T["FPf"][j, m - 1] > fp_limit or T["FNnf"][j] + T["FNf"][j, 0] > fn_limit:
            continue                                   # infeasible even at the extremes
        l = 0
        while l + 1 < m and int(T["FNnf"][j]) + int(T["FNf"][j, l + 1]) <= fn_limit:
            l += 1
        h = m - 1
        while h - 1 >= 0 and int(T["FPnf"][j]) + int(T["FPf"][j, h - 1]) <= fp_limit:
            h -= 1
        if l > h:
            best_k = min(range(h, l + 1), key=lambda t: (triple_counts(T, j, t, t)[3], -t, t))
            l = h = best_k
        fp, fn, F, U = triple_counts(T, j, l, h)
        cands.append(((cost_ps(T["checked"], F, U, t_mse, t_snn, t_full), U, j, -l, h),
                      dict(j=j, l=l, h=h, fp=fp, fn=fn, F=F, U=U,
                           cost=cost_ps(T["checked"], F, U, t_mse, t_snn, t_full))))
    if not cands:
        return None
    return min(cands, key=lambda c: c[0])[1]


# --------------------------------------------------------------------------
# N1 DD fitting — P:557-558 "computes the reference image
#    by averaging frames where the reference model returns no labels";
#    P:577-581 / P:850-853 "trains a logistic regression (LR) classifier to weigh
#    each block"; SPEC build_reference_image S:134-142, train_block_weights
#    S:209-217.  Readings: R-21 rounding half up, on the 50x50 small
#    frames the DD compares; R-22 LR = the minimiser of the mean log loss
#    (+ l2/2 |w|^2, l2 > 0) over z-scored features (Newton's method to a gradient
#    tolerance), folded back to raw features.
# --------------------------------------------------------------------------
def reference_image(small: np.ndarray, labels: np.ndarray) -> np.ndarray:
    """small uint8 [n, h, w, 3], labels [n] (0 = no object).  Per-pixel mean over
    the negative frames, rounded half up: floor((2*S + m) / (2*m)), m = #negatives.
    Raises ValueError when there is no negative frame (caller falls back
    to earlier-frame mode)."""
    neg = np.asarray(labels) == 0
    m = int(neg.sum())
    if m == 0:
        raise ValueError("no negative frame: use the earlier-frame difference detector")
    S = small[neg].astype(np.int64).sum(axis=0)
    return ((2 * S + m) // (2 * m)).astype(np.uint8)


def block_features(small: np.ndarray, grid: int, mode: int, ref=None, k: int = 0) -> np.ndarray:
    """float64 [n, grid*grid]: row i = blocked_mse(frame i, anchor) (O3), anchor =
    the reference image (mode 0) or frame i - k of the same batch (mode 1; rows
    i < k have no anchor and are NaN)."""
    n = small.shape[0]
    out = np.full((n, grid * grid), np.nan)
    for i in range(n):
        if mode == 0:
            out[i] = blocked_mse(small[i], ref, grid)
        elif i >= k:
            out[i] = blocked_mse(small[i], small[i - k], grid)
    return out


LR_STEP_LADDER = [2.0 ** -i for i in range(16)]     # backtracking steps 1, 1/2, ..., 2^-15
LR_ARMIJO_C = 1e-4


def lr_objective(X, t, v, l2: float) -> float:
    """J(w, b) = mean_i [softplus(z_i) - t_i z_i] + l2/2 |w|^2,  z = X w + b (X z-scored)."""
    z = X @ v[:-1] + v[-1]
    return float(np.mean(np.logaddexp(0.0, z) - t * z) + 0.5 * l2 * np.dot(v[:-1], v[:-1]))


def lr_fit(F: np.ndarray, t: np.ndarray, l2: float | None = None, tol: float = 1e-9, max_iters: int = 100,
           info: dict | None = None):
    """Logistic regression (R-22), fp64: the minimiser of
        J(w, b) = mean_i [log(1 + exp(z_i)) - t_i z_i] + l2/2 |w|^2,   z_i = x_i . w + b,
    x_i = (F_i - mu) / sd per feature (population mean / std; constant features sd := 1).
    l2 > 0 (default 1/n: scikit-learn's C = 1 written per example, P:850-851 names
    scikit-learn) makes J strictly convex, so the minimiser exists and is unique even on
    separable data.  Found by Newton's method from v = (w, b) = 0; each iteration:
        p = sigmoid(z);  g = [X^T (p - t) / n + l2 w ;  mean(p - t)]
        stop if max|g| <= tol
        H = [X 1]^T diag(p (1 - p)) [X 1] / n + l2 diag(1, .., 1, 0)
        Delta = -H^{-1} g                                  (Cholesky solve)
        s = first of 1, 1/2, ..., 2^-15 with J(v + s Delta) <= J(v) + 1e-4 s g.Delta
            (Armijo backtracking); if none, stop (the rounding floor is reached)
        v = v + s Delta
    Returns raw-feature parameters (w / sd, b - sum(w * mu / sd)) so that the scorer's
    logit b + sum_k w_k m_k equals the fitted model's.  info (optional dict) receives
    iters, grad_inf (max|g| at the returned point) and J.  Errors: n < 2 or one class
    only ("advising global metric"), l2 <= 0."""
    F = np.asarray(F, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    n, d = F.shape
    if n < 2 or t.min() == t.max():
        raise ValueError("LR fit needs >= 2 examples of both classes; use the global metric")
    if l2 is None:
        l2 = 1.0 / n
    if not l2 > 0:
        raise ValueError("l2 must be > 0 (a minimiser must exist)")
    mu = F.mean(axis=0)
    sd = F.std(axis=0)
    sd = np.where(sd > 0, sd, 1.0)
    X = (F - mu) / sd
    X1 = np.hstack([X, np.ones((n, 1))])
    reg = np.full(d + 1, l2)
    reg[d] = 0.0
    v = np.zeros(d + 1)
    it = 0
    while True:
        p = 1.0 / (1.0 + np.exp(-(X1 @ v)))
        g = X1.T @ (p - t) / n + reg * v
        if np.max(np.abs(g)) <= tol or it >= max_iters:
            break
        H = (X1 * (p * (1.0 - p))[:, None]).T @ X1 / n + np.diag(reg)
        L = np.linalg.cholesky(H)
        delta = -np.linalg.solve(L.T, np.linalg.solve(L, g))
        J0, slope = lr_objective(X, t, v, l2), float(g @ delta)
        step = next((s for s in LR_STEP_LADDER
                     if lr_objective(X, t, v + s * delta, l2) <= J0 + LR_ARMIJO_C * s * slope), None)
        if step is None:
            break
        v = v + step * delta
        it += 1
    if info is not None:
        info.update(iters=it, grad_inf=float(np.max(np.abs(g))), J=lr_objective(X, t, v, l2))
    w = v[:d]
    return w / sd, v[d] - float(np.sum(w * mu / sd))


def lr_loss(F, t, w_raw, b_raw, l2: float = 0.0) -> float:
    """Mean log loss of raw-feature parameters (+ l2/2 |w_std|^2 in the z-scored
    parameterisation), the objective lr_fit descends (used by its pins)."""
    F = np.asarray(F, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    sd = F.std(axis=0)
    sd = np.where(sd > 0, sd, 1.0)
    z = F @ w_raw + b_raw
    loss = np.mean(np.logaddexp(0.0, z) - t * z)
    return float(loss + 0.5 * l2 * np.sum((w_raw * sd) ** 2))


# --------------------------------------------------------------------------
# N2 Full CBO search — P:717-779 "NoScope's CBO ...
#    profiles each filter ... on the evaluation set ... sweeps delta_diff ... the
#    cost model selects the cheapest cascade meeting FP*/FN*" over the DD
#    configurations x specialized-NN architectures.
#    Reading R-23: every DD config and every CNN runs unfiltered on
#    all evaluation frames; one sweep per (DD, CNN) pair with that CNN's own
#    T_SNN; overall argmin of (infeasible, violation, cost, U, dd, cnn).
# --------------------------------------------------------------------------
def cbo_search(small: np.ndarray, y: np.ndarray, dd_cfgs, delta_grids, cnns, u, t_mse: int,
               t_full: int, fp_limit: int, fn_limit: int):
    """small uint8 [n, h, w, 3] (evaluation split, downsampled); dd_cfgs: list of
    DDConfig; delta_grids: their candidate arrays; cnns: list of (arch, weights,
    t_snn_ps).  Returns (dd index, cnn index, sweep_best dict of that pair)."""
    logits = [cnn_logits(small, arch, w) for arch, w, _ in cnns]
    best, best_key = None, None
    for di, cfg in enumerate(dd_cfgs):
        s, _ = diff_detect(small, cfg)
        a = build_records(s, y, cfg.mode, cfg.t_diff_frames)
        for ci, (_, _, t_snn) in enumerate(cnns):
            _, b = sweep(s, logits[ci], y, a, delta_grids[di], u, (t_mse, t_snn, t_full),
                         fp_limit, fn_limit)
            viol = 0 if b["feasible"] else max(b["fp"] - fp_limit, b["fn"] - fn_limit, 0)
            key = (0 if b["feasible"] else 1, viol, b["cost"], b["U"], di, ci)
            if best_key is None or key < best_key:
                best, best_key = (di, ci, b), key
    return best


# --------------------------------------------------------------------------
# N3 Evaluation harness — P:1027-1032 "comparing frames
#    labeled by the reference model and NoScope in 30 frame windows ... agree on
#    the presence of the target object in 28 of the 30 frames"
#    factor analysis / lesion study.  Reading R-24:
#    the modeled cost charges T_MSE per checked frame only when the difference
#    detector is in the cascade, T_SNN per fired frame only when the specialized
#    NN is, and T_full per frame that reaches the reference NN.
# --------------------------------------------------------------------------
def windowed_accuracy(pred, ref, window: int = 30, agree_min: int = 28) -> float:
    """Consecutive non-overlapping windows (final partial window dropped); a
    window is correct iff >= agree_min frames agree."""
    pred, ref = np.asarray(pred), np.asarray(ref)
    if pred.shape != ref.shape:
        raise ValueError("length mismatch")
    nw = len(pred) // window
    if nw == 0:
        raise ValueError("shorter than one window")
    agree = (pred[:nw * window] != 0) == (ref[:nw * window] != 0)
    per = agree.reshape(nw, window).sum(axis=1)
    return float((per >= agree_min).sum()) / nw


def fp_fn(pred, ref):
    """(fp, fn, tp, tn) frame counts."""
    p, r = np.asarray(pred) != 0, np.asarray(ref) != 0
    if p.shape != r.shape:
        raise ValueError("length mismatch")
    return int((p & ~r).sum()), int((~p & r).sum()), int((p & r).sum()), int((~p & ~r).sum())


def cascade_counts(res) -> dict:
    """Per-stage frame counts of one oracle cascade result."""
    disp, route_pf = res["disp"], res["route"]
    return dict(n=len(disp), checked=int((disp != SKIPPED).sum()), fired=int((disp == FIRED).sum()),
                uncertain=int((route_pf == R_UNC).sum()))


def modeled_speedup(c: dict, stages, t_mse: int, t_snn: int, t_full: int) -> float:
    """N*T_full / modeled cascade time (R-24).  stages: subset of
    {"skip", "dd", "cnn"}; frames reaching the reference NN = uncertain frames
    with the CNN, fired frames without it."""
    oracle_frames = c["uncertain"] if "cnn" in stages else c["fired"]
    t = (c["checked"] * t_mse if "dd" in stages else 0) + (c["fired"] * t_snn if "cnn" in stages else 0) \
        + oracle_frames * t_full
    if t == 0:
        raise ValueError("zero modeled time")
    return c["n"] * t_full / t


FACTOR_ROWS = [("oracle only", ()), ("+skipping", ("skip",)), ("+difference detection", ("skip", "dd")),
               ("+specialized model", ("skip", "dd", "cnn"))]
LESION_ROWS = [("full", ("skip", "dd", "cnn")), ("-skipping", ("dd", "cnn")),
               ("-difference detection", ("skip", "cnn")), ("-specialized model", ("skip", "dd"))]


def stage_config(cfg: DDConfig, lo: float, hi: float, stages):
    """The cascade with only `stages` active: no skipping -> t_skip 1; no DD ->
    delta = -inf (every checked frame fires); no CNN -> (lo, hi) = (-inf, +inf)
    (every fired frame is uncertain and goes to the reference NN)."""
    c = dataclasses.replace(cfg, t_skip_frames=cfg.t_skip_frames if "skip" in stages else 1,
                            delta_diff=cfg.delta_diff if "dd" in stages else -math.inf)
    return c, (lo if "cnn" in stages else -math.inf), (hi if "cnn" in stages else math.inf)


def factor_analysis(frames_hw3, cfg: DDConfig, arch, weights, lo, hi, truth, timing, rows=FACTOR_ROWS):
    """Rows of (name, windowed accuracy vs the reference labels, fp, fn, counts,
    modeled speedup) for nested (FACTOR_ROWS) or leave-one-out (LESION_ROWS)
    stage sets."""
    out = []
    for name, stages in rows:
        c, l, h = stage_config(cfg, lo, hi, stages)
        res = cascade(frames_hw3, c, arch, weights, l, h, truth)
        cnt = cascade_counts(res)
        fp, fn, _, _ = fp_fn(res["labels"], truth)
        out.append(dict(name=name, accuracy=windowed_accuracy(res["labels"], truth), fp=fp, fn=fn,
                        speedup=modeled_speedup(cnt, stages, *timing), **cnt))
    return out


# --------------------------------------------------------------------------
# N4 Specialized-CNN training — P:472-477 "We train our
#    specialized NNs ... RMSprop ... between one and five epochs ... early
#    stopping", P:855-860 (cross-validation set).  Reading R-25:
#    fp64 here / fp32 on the GPU, no bf16 rounding inside training (the input is
#    the inference normalisation O6); mean binary cross-entropy on the logit;
#    RMSprop v <- rho v + (1 - rho) g^2, w <- w - lr g / (sqrt(v) + eps); the
#    mini-batch order is an input (a permutation per epoch); max-pool gradients go
#    to the first maximum of each window in (dy, dx) row-major order; stop after
#    the first epoch whose training loss rose, return the best
#    cross-validation epoch.
# --------------------------------------------------------------------------
def cnn_params_from_weights(weights: dict) -> dict:
    """bf16-bit weight dict (synthgen layout) -> fp64 parameter dict."""
    return {"conv_w": [bf16_bits_to_f64(w) for w in weights["conv_w"]],
            "conv_b": [np.asarray(b, np.float64) for b in weights["conv_b"]],
            "fc1_w": bf16_bits_to_f64(weights["fc1_w"]), "fc1_b": np.asarray(weights["fc1_b"], np.float64),
            "fc2_w": bf16_bits_to_f64(weights["fc2_w"]), "fc2_b": np.asarray(weights["fc2_b"], np.float64)}


def _pool_argmax(a: np.ndarray):
    """2x2 floor max pool returning (pooled, index 0..3 of the first maximum)."""
    n, H, W, C = a.shape
    Ho, Wo = H // 2, W // 2
    v = a[:, :2 * Ho, :2 * Wo, :].reshape(n, Ho, 2, Wo, 2, C).transpose(0, 1, 3, 2, 4, 5)
    v = v.reshape(n, Ho, Wo, 4, C)                     # window member q = 2*dy + dx
    return v.max(axis=3), v.argmax(axis=3)             # argmax: first maximum


def cnn_forward_train(small: np.ndarray, arch, P: dict):
    """Forward pass keeping what the backward pass needs (fp64, no bf16)."""
    x = normalize_input(small, arch.chan_mean)
    cache = []
    for l in range(arch.n_conv):
        pre = conv3x3_same(x, P["conv_w"][l], P["conv_b"][l])
        a = np.maximum(pre, 0.0)
        p, arg = _pool_argmax(a)
        cache.append((x, a, arg))
        x = p
    f = x.reshape(x.shape[0], -1)
    h1 = np.maximum(f @ P["fc1_w"].T + P["fc1_b"], 0.0)
    z = h1 @ P["fc2_w"] + P["fc2_b"][0]
    return z, (cache, x.shape, f, h1)


def bce_with_logits(z, t) -> float:
    """mean(softplus(z) - t z)."""
    return float(np.mean(np.logaddexp(0.0, z) - np.asarray(t, np.float64) * z))


def cnn_backward(z, t, st, P: dict) -> dict:
    """Gradients of the mean BCE w.r.t. every parameter (same keys as P)."""
    cache, xs, f, h1 = st
    B = len(z)
    dz = (1.0 / (1.0 + np.exp(-z)) - np.asarray(t, np.float64)) / B
    g = {"fc2_w": h1.T @ dz, "fc2_b": np.array([dz.sum()])}
    dh1 = np.outer(dz, P["fc2_w"]) * (h1 > 0)
    g["fc1_w"] = dh1.T @ f
    g["fc1_b"] = dh1.sum(axis=0)
    dx = (dh1 @ P["fc1_w"]).reshape(xs)
    g["conv_w"] = [None] * len(cache)
    g["conv_b"] = [None] * len(cache)
    for l in range(len(cache) - 1, -1, -1):
        x, a, arg = cache[l]
        n, H, W, C = a.shape
        Ho, Wo = H // 2, W // 2
        da = np.zeros_like(a)
        onehot = np.eye(4)[arg]                                        # [n, Ho, Wo, C, 4]
        d4 = (onehot * dx[..., None]).transpose(0, 1, 2, 4, 3).reshape(n, Ho, Wo, 2, 2, C)
        da[:, :2 * Ho, :2 * Wo, :] = d4.transpose(0, 1, 3, 2, 4, 5).reshape(n, 2 * Ho, 2 * Wo, C)
        da *= (a > 0)
        cin = x.shape[3]
        xp = np.zeros((n, H + 2, W + 2, cin))
        xp[:, 1:H + 1, 1:W + 1, :] = x
        gw = np.empty((C, 3, 3, cin))
        for ky in range(3):
            for kx in range(3):
                gw[:, ky, kx, :] = da.reshape(-1, C).T @ xp[:, ky:ky + H, kx:kx + W, :].reshape(-1, cin)
        g["conv_w"][l] = gw
        g["conv_b"][l] = da.sum(axis=(0, 1, 2))
        if l > 0:
            dap = np.zeros((n, H + 2, W + 2, C))
            dap[:, 1:H + 1, 1:W + 1, :] = da
            dxl = np.zeros((n, H, W, cin))
            w = P["conv_w"][l]
            for ky in range(3):
                for kx in range(3):   # x[y+ky-1] fed out[y] => dx[y'] += da[y'-ky+1] w[ky]
                    dxl += dap[:, 2 - ky:2 - ky + H, 2 - kx:2 - kx + W, :] @ w[:, ky, kx, :]
            dx = dxl
    return g


def rmsprop_step(P: dict, G: dict, V: dict, lr: float, rho: float, eps: float):
    """v <- rho v + (1 - rho) g^2; p <- p - lr g / (sqrt(v) + eps), every tensor."""
    def upd(p, g, v):
        v[...] = rho * v + (1.0 - rho) * g * g
        p[...] = p - lr * g / (np.sqrt(v) + eps)
    for k in ("conv_w", "conv_b"):
        for l in range(len(P[k])):
            upd(P[k][l], G[k][l], V[k][l])
    for k in ("fc1_w", "fc1_b", "fc2_w", "fc2_b"):
        upd(P[k], G[k], V[k])


def _zeros_like_params(P):
    return {k: ([np.zeros_like(x) for x in v] if isinstance(v, list) else np.zeros_like(v)) for k, v in P.items()}


def _copy_params(P):
    return {k: ([x.copy() for x in v] if isinstance(v, list) else v.copy()) for k, v in P.items()}


def train_should_stop(hist) -> bool:
    """P:474-475 "early stopping if the training loss increases" ("stops early
    when epoch-end training loss exceeds the previous epoch's"): after epoch e >= 1,
    stop iff train_loss[e] > train_loss[e - 1] (strict)."""
    e = len(hist) - 1
    if e > 0 and hist[e][0] > hist[e - 1][0]:
        return True
    return False


def cnn_train(small_tr, y_tr, small_va, y_va, arch, P0: dict, perms, batch: int, lr=1e-3, rho=0.9,
              eps=1e-7):
    """RMSprop over at most len(perms) epochs (the paper's 1-5); epoch e visits
    perms[e] in mini-batches of `batch` (last one partial).  The epoch's training loss is
    the mean over its samples of the loss of their batch before that batch's update
    (Keras's reported epoch loss; P:472 names Keras).  After each epoch the
    cross-validation loss is recorded; training stops after the first epoch whose
    training loss exceeds the previous epoch's (train_should_stop), and the parameters
    of the epoch with the lowest cross-validation loss (earliest on ties) are returned
    (S:317).  Returns (params, history) with history = [(train_loss, val_loss)] per
    epoch run."""
    P = _copy_params(P0)
    V = _zeros_like_params(P)
    best, best_val, hist = _copy_params(P), math.inf, []
    for perm in perms:
        tot = 0.0
        for s in range(0, len(perm), batch):
            idx = np.asarray(perm[s:s + batch])
            z, st = cnn_forward_train(small_tr[idx], arch, P)
            tot += bce_with_logits(z, y_tr[idx]) * len(idx)
            rmsprop_step(P, cnn_backward(z, y_tr[idx], st, P), V, lr, rho, eps)
        zv, _ = cnn_forward_train(small_va, arch, P)
        val = bce_with_logits(zv, y_va)
        hist.append((tot / len(perm), val))
        if val < best_val:
            best, best_val = _copy_params(P), val
        if train_should_stop(hist):
            break
    return best, hist
