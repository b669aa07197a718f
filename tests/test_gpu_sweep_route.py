"""GPU parity: routing (bit-exact on identical logits) and the CBO threshold
sweep (tables and best triple bit-exact vs the oracle; sampled entries and
optimality properties at the 1M-record BASELINE size)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import ns, requires_gpu

pytestmark = [pytest.mark.gpu, requires_gpu]


@pytest.mark.parametrize("n", [0, 1, 100, 4096, 4097, 50001])
def test_route_bit_exact(n):
    nsm = ns()
    rng = np.random.default_rng(n)
    z = rng.normal(0, 2, n).astype(np.float32)
    if n > 10:
        z[:5] = np.float32([-1.0, 1.0, -1.0, 1.0, 0.5])   # exact ties at lo / hi
    for lo, hi in [(-1.0, 1.0), (-math.inf, math.inf), (0.5, 0.5), (-math.inf, -1.0)]:
        r, unc, nunc = nsm.noscope_route_logits(lo, hi, torch.from_numpy(z).cuda())
        torch.cuda.synchronize()
        ro = O.route(z, lo, hi)
        assert np.array_equal(r.cpu().numpy(), ro)
        k = int(nunc.item())
        assert np.array_equal(unc.cpu().numpy()[:k], np.flatnonzero(ro == O.R_UNC))


def _gpu_sweep(nsm, s, z, y, a, delta, u, timing, fpl, fnl, split=1):
    dev = "cuda"
    T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).to(dev)
    dd, uu = T(delta, np.float64), T(u, np.float32)
    hist = torch.zeros(nsm.sweep_hist_words(len(delta), len(u)), dtype=torch.int64, device=dev)
    bounds = np.linspace(0, len(s), split + 1).astype(int)
    for i in range(split):                         # phase 1 accumulates (as after an allreduce)
        sl = slice(bounds[i], bounds[i + 1])
        nsm.noscope_threshold_sweep(1, T(s[sl], np.float64), T(z[sl], np.float32),
                                    T(y[sl], np.uint8), T(a[sl], np.uint8), dd, uu, hist)
    nd, m = len(delta), len(u)
    tabs = {k: torch.zeros(nd * (m if k in ("FPf", "FNf", "GE", "GT") else 1), dtype=torch.int64,
                           device=dev) for k in ("F", "FPnf", "FNnf", "FPf", "FNf", "GE", "GT")}
    best, code = nsm.noscope_threshold_sweep(2, None, None, None, None, dd, uu, hist, timing,
                                             fpl, fnl, tables=tabs)
    return best, code, {k: v.cpu().numpy().astype(np.uint64) for k, v in tabs.items()}, hist


@pytest.mark.parametrize("seed", range(40))
def test_sweep_random_instances_bit_exact(seed):
    nsm = ns()
    n = [1, 7, 60, 300, 999][seed % 5]
    s, z, y, a, delta, u = sg.random_sweep_records(n, seed + 1000, n_delta=9, m=8)
    timing = [(1, 10, 1000), (3, 5, 7)][seed % 2]
    fpl, fnl = seed % 3, (seed // 3) % 3
    T, best_o = O.sweep(s, z, y, a, delta, u, timing, fpl, fnl)
    best, code, tabs, _ = _gpu_sweep(nsm, s, z, y, a, delta, u, timing, fpl, fnl, split=1 + seed % 3)
    for k in ("F", "FPnf", "FNnf"):
        assert np.array_equal(tabs[k], T[k]), k
    for k in ("FPf", "FNf", "GE", "GT"):
        assert np.array_equal(tabs[k].reshape(len(delta), len(u)), T[k]), k
    assert (code == 7) == (not best_o["feasible"])
    for k_g, k_o in [("j", "j"), ("l", "l"), ("h", "h"), ("fp", "fp"), ("fn", "fn"),
                     ("uncertain", "U"), ("fired", "F"), ("cost_ps", "cost")]:
        assert best[k_g] == best_o[k_o], (k_g, best, best_o)
    assert best["checked"] == T["checked"] and best["total"] == len(s)


def test_sweep_spec_six_frame_instance():
    nsm = ns()
    s = np.array([9, 8, 5, 4, 2, 1], np.float64)
    y = np.array([1, 1, 0, 1, 0, 0], np.uint8)
    c = np.array([.95, .9, .6, .55, .2, .1])
    z = np.log(c / (1 - c)).astype(np.float32)
    a = np.zeros(6, np.uint8)
    delta = np.array([-np.inf, 0.5, 1.5, 3, 4.5, 6.5, 8.5, 9.5])
    u = np.unique(np.concatenate([[-np.inf, np.inf], z])).astype(np.float32)
    bf = O.sweep_brute_force(s, z, y, a, delta, u, (1, 10, 1000), 1, 1)
    best, code, _, _ = _gpu_sweep(nsm, s, z, y, a, delta, u, (1, 10, 1000), 1, 1)
    assert code == 0 and (best["j"], best["l"], best["h"]) == (bf["j"], bf["l"], bf["h"])


def test_sweep_1m_records_sampled():
    """BASELINE configs[3] size: 1M records, 100 x 100 candidates; sampled table
    entries recomputed one by one with the oracle definition, best triple's counts
    re-derived, and optimality checked against random feasible triples."""
    nsm = ns()
    rng = np.random.default_rng(77)
    N = 1_000_000
    y = (rng.random(N) < 0.15).astype(np.uint8)
    s = np.where(rng.random(N) < 0.1, -np.inf, rng.gamma(2.0, 10.0, N) + 40.0 * y)
    z = (rng.normal(0, 1, N) + 2.5 * y - 1.0).astype(np.float32)
    a = np.where(np.isinf(s), y, 0).astype(np.uint8)
    delta = sg.delta_grid(s, 100)
    u = sg.logit_grid(100)
    timing = (1_000, 20_000, 12_500_000)
    lim = N // 100
    best, code, tabs, hist = _gpu_sweep(nsm, s, z, y, a, delta, u, timing, lim, lim, split=4)
    nd, m = len(delta), len(u)
    for j in rng.integers(0, nd, 6):
        fired = s > delta[j]
        assert tabs["F"][j] == fired.sum()
        assert tabs["FPnf"][j] == (~fired & (a == 1) & (y == 0)).sum()
        for h in rng.integers(0, m, 3):
            assert tabs["FPf"].reshape(nd, m)[j, h] == (fired & (z > u[h]) & (y == 0)).sum()
            assert tabs["GE"].reshape(nd, m)[j, h] == (fired & (z >= u[h])).sum()
            assert tabs["FNf"].reshape(nd, m)[j, h] == (fired & (z < u[h]) & (y == 1)).sum()
    assert code == 0
    j, l, h = best["j"], best["l"], best["h"]
    fired = s > delta[j]
    out = np.where(fired, np.where(z < u[l], 0, np.where(z > u[h], 1, y)), a)
    assert best["fp"] == ((out == 1) & (y == 0)).sum() <= lim
    assert best["fn"] == ((out == 0) & (y == 1)).sum() <= lim
    U = int((fired & (z >= u[l]) & (z <= u[h])).sum())
    assert best["uncertain"] == U
    checked = int(np.isfinite(s).sum() + (s == np.inf).sum())
    assert best["cost_ps"] == checked * timing[0] + int(fired.sum()) * timing[1] + U * timing[2]
    T = {k: (tabs[k].reshape(nd, m) if k in ("FPf", "FNf", "GE", "GT") else tabs[k]) for k in tabs}
    T["checked"] = checked
    for _ in range(2000):
        jj = int(rng.integers(0, nd)); ll = int(rng.integers(0, m)); hh = int(rng.integers(ll, m))
        fp, fn, F, UU = O.triple_counts(T, jj, ll, hh)
        if fp <= lim and fn <= lim:
            assert O.cost_ps(checked, F, UU, *timing) >= best["cost_ps"]


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 4095, 4096, 4097, 100003])
@pytest.mark.parametrize("t_skip,seg", [(1, 0), (3, 7), (15, 0)])
def test_compact_fired_bit_exact(n, t_skip, seg):
    """H4 stable compaction (+ the t_skip rewrite) vs the oracle's O5 loop, on the
    aligned (16-byte vector) and misaligned (scalar) load paths."""
    nsm = ns()
    rng = np.random.default_rng(n * 31 + t_skip)
    disp = rng.choice([O.SUPPRESSED, O.FIRED], size=n, p=[0.85, 0.15]).astype(np.uint8)
    want = disp.copy()
    tau = seg + np.arange(n)
    want[tau % t_skip != 0] = O.SKIPPED
    want_idx = O.compact(want)
    for off in (0, 1):
        buf = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
        d = buf[off:off + n]
        d.copy_(torch.from_numpy(disp))
        idx, cnt = nsm.noscope_compact_fired(d, seg_offset=seg, t_skip=t_skip)
        torch.cuda.synchronize()
        k = int(cnt.item())
        assert k == len(want_idx)
        assert np.array_equal(idx.cpu().numpy()[:k], want_idx)
        assert np.array_equal(d.cpu().numpy(), want)


@pytest.mark.parametrize("t_skip", [1, 3])
def test_compact_fired_multi_window(t_skip):
    """More than one 64 MB compaction window (8,192 tiles of 8,192 frames): the running
    offset carried across windows, ragged tail; checked against numpy.flatnonzero (the
    O5 pin) on 70,000,123 dispositions."""
    nsm = ns()
    n = 70_000_123
    g = torch.Generator(device="cuda").manual_seed(17)
    d = torch.where(torch.rand(n, device="cuda", generator=g) < 0.15,
                    torch.full((), O.FIRED, dtype=torch.uint8, device="cuda"),
                    torch.full((), O.SUPPRESSED, dtype=torch.uint8, device="cuda"))
    disp = d.cpu().numpy()
    want = disp.copy()
    want[(5 + np.arange(n)) % t_skip != 0] = O.SKIPPED
    idx, cnt = nsm.noscope_compact_fired(d, seg_offset=5, t_skip=t_skip)
    torch.cuda.synchronize()
    ref = np.flatnonzero(want == O.FIRED)
    k = int(cnt.item())
    assert k == len(ref)
    assert np.array_equal(idx[:k].cpu().numpy(), ref)
    assert np.array_equal(d.cpu().numpy(), want)


def _best_by_tables(T, timing, fpl, fnl):
    """Lexicographic argmin of (cost, U, j, -l, h) over feasible l <= h, from the
    oracle's tables, vectorised over (l, h) per j (O9's objective restated)."""
    nd, m = T["FPf"].shape
    t_mse, t_snn, t_full = timing
    best = None
    li, hi = np.triu_indices(m)
    for j in range(nd):
        fp = int(T["FPnf"][j]) + T["FPf"][j].astype(np.int64)[hi]
        fn = int(T["FNnf"][j]) + T["FNf"][j].astype(np.int64)[li]
        U = T["GE"][j].astype(np.int64)[li] - T["GT"][j].astype(np.int64)[hi]
        ok = (fp <= fpl) & (fn <= fnl)
        if not ok.any():
            continue
        cost = T["checked"] * t_mse + int(T["F"][j]) * t_snn + U * t_full
        o = np.lexsort((hi[ok], -li[ok], U[ok], cost[ok]))[0]
        key = (int(cost[ok][o]), int(U[ok][o]), j, -int(li[ok][o]), int(hi[ok][o]))
        if best is None or key < best:
            best = key
    return best


@pytest.mark.parametrize("nd,m,n", [(40, 2048, 3000), (2000, 8, 5000),
                                    (3, 1, 2000), (7, 33, 4000), (5, 63, 4000), (4, 1001, 3000),
                                    (3, 1024, 3000), (100, 101, 20000), (64, 127, 5000), (127, 64, 5000),
                                    (200, 255, 5000), (7, 7, 3000), (1000, 1000, 3000)])
def test_sweep_candidate_limits(nd, m, n):
    """m = 2048 (the largest accepted candidate count: phase 2's per-delta tables
    use 164 KB of shared memory) and nd = 2,000 (the d-suffix pass is O(nd*m)); and
    the evaluation's work split (row pairs {l, m-1-l} dealt to P = (m+1)//32 lanes,
    1..32): one candidate, odd m (a self-paired middle row) with P = 1, 2 and 31, even
    m with P = 32; and the histogram's fixed-depth instantiations (equal depths 3..11:
    depth 7 = 64..127 candidates, the 100-candidate grids, at both ends of its range;
    depths 8, 3 and 10)."""
    nsm = ns()
    s, z, y, a, _, _ = sg.random_sweep_records(n, 77)
    delta = np.linspace(-7.0, 7.0, nd)                          # distinct, sorted
    u = np.linspace(-7.0, 7.0, m).astype(np.float32)
    assert len(np.unique(u)) == m
    rng = np.random.default_rng(5)
    hs, hz = rng.random(n) < 0.2, rng.random(n) < 0.2           # exact candidate hits (ties)
    s[hs] = rng.choice(delta, int(hs.sum()))
    z[hz] = rng.choice(u, int(hz.sum()))
    timing = (1, 10, 1000)
    fpl, fnl = n // 20, n // 20
    T = O.sweep_tables(s, z, y, a, delta, u)
    best, code, tabs, _ = _gpu_sweep(nsm, s, z, y, a, delta, u, timing, fpl, fnl, split=2)
    for k in ("F", "FPnf", "FNnf"):
        assert np.array_equal(tabs[k], T[k]), k
    for k in ("FPf", "FNf", "GE", "GT"):
        assert np.array_equal(tabs[k].reshape(nd, m), T[k]), k
    key = _best_by_tables(T, timing, fpl, fnl)
    if key is None:   # no feasible triple (m = 1): the least-violating one, from the oracle's O9
        _, best_o = O.sweep(s, z, y, a, delta, u, timing, fpl, fnl)
        assert code == 7 and not best_o["feasible"]
        assert (best["j"], best["l"], best["h"], best["cost_ps"]) == \
            (best_o["j"], best_o["l"], best_o["h"], best_o["cost"])
        return
    assert code == 0
    assert (best["cost_ps"], best["uncertain"], best["j"], -best["l"], best["h"]) == key


@pytest.mark.parametrize("mode,k,t_skip", [(0, 1, 1), (1, 30, 1), (1, 7, 3), (0, 1, 15), (1, 4, 4)])
def test_sweep_records_a_matches_oracle(mode, k, t_skip):
    """The a[] record column (label emitted when not fired) == O.build_records."""
    nsm = ns()
    n = 5003
    rng = np.random.default_rng(k * 31 + t_skip)
    s = rng.normal(0, 1, n)
    s[np.arange(n) % t_skip != 0] = -np.inf
    s[:k][np.arange(min(k, n)) % t_skip == 0] = np.inf if mode == 1 else s[:k][np.arange(min(k, n)) % t_skip == 0]
    y = (rng.random(n) < 0.3).astype(np.uint8)
    a = nsm.noscope_sweep_records(torch.from_numpy(s).cuda(), torch.from_numpy(y).cuda(), mode, k, t_skip)
    torch.cuda.synchronize()
    assert np.array_equal(a.cpu().numpy(), O.build_records(s, y, mode, k))


@pytest.mark.parametrize("p_fired", [0.0, 1.0, 0.5])
def test_compact_fired_densities_many_ctas(p_fired):
    """None / all / half fired over 3,000,017 frames (733 warp-chunks: every CTA of
    the persistent grid owns a range; the all-fired case writes one index per frame)."""
    nsm = ns()
    n = 3_000_017
    g = torch.Generator(device="cuda").manual_seed(3)
    d = torch.where(torch.rand(n, device="cuda", generator=g) < p_fired,
                    torch.full((), O.FIRED, dtype=torch.uint8, device="cuda"),
                    torch.full((), O.SUPPRESSED, dtype=torch.uint8, device="cuda"))
    idx, cnt = nsm.noscope_compact_fired(d)
    torch.cuda.synchronize()
    ref = np.flatnonzero(d.cpu().numpy() == O.FIRED)
    k = int(cnt.item())
    assert k == len(ref) and np.array_equal(idx[:k].cpu().numpy(), ref)


def test_route_many_ctas_vs_numpy():
    """2^24 + 13 logits (every CTA of the persistent grid busy, ragged tail) with exact
    ties at the thresholds; codes and the uncertain list vs the O7 definition in numpy."""
    nsm = ns()
    n = (1 << 24) + 13
    g = torch.Generator(device="cuda").manual_seed(9)
    z = torch.randn(n, device="cuda", generator=g)
    z[::1001] = 0.5
    z[7::997] = -0.25
    lo, hi = -0.25, 0.5
    r, unc, nunc = nsm.noscope_route_logits(lo, hi, z)
    torch.cuda.synchronize()
    zn = z.cpu().numpy()
    ro = np.where(zn < np.float32(lo), O.R_NEG, np.where(zn > np.float32(hi), O.R_POS, O.R_UNC)).astype(np.uint8)
    assert np.array_equal(r.cpu().numpy(), ro)
    k = int(nunc.item())
    assert np.array_equal(unc[:k].cpu().numpy(), np.flatnonzero(ro == O.R_UNC))


def test_sweep_async_phase2_matches_sync():
    """NOSCOPE_SWEEP_ASYNC: phase 2 copies the best triple into page-locked memory
    without synchronising; after the stream completes it equals the synchronous result."""
    nsm = ns()
    s, z, y, a, delta, u = sg.random_sweep_records(5000, 11, n_delta=20, m=16)
    T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()
    args = (T(s, np.float64), T(z, np.float32), T(y, np.uint8), T(a, np.uint8), T(delta, np.float64),
            T(u, np.float32))
    words = nsm.sweep_hist_words(len(delta), len(u))
    h1 = torch.zeros(words, dtype=torch.int64, device="cuda")
    best_sync, code = nsm.noscope_threshold_sweep(3, *args, h1, (1, 10, 1000), 200, 200)
    h2 = torch.zeros(words, dtype=torch.int64, device="cuda")
    out = nsm.pinned_sweep_best()
    r, code2 = nsm.noscope_threshold_sweep(3, *args, h2, (1, 10, 1000), 200, 200, best_out=out)
    torch.cuda.synchronize()
    assert code2 == 0 and nsm.sweep_best_dict(out) == best_sync


@pytest.mark.parametrize("m,seed", [(33, 1), (63, 2), (64, 3), (65, 4)])
def test_sweep_eval_split_infeasible_and_feasible(m, seed):
    """The least-violating (no feasible triple) and the feasible argmin at odd and even m
    across the evaluation's work-split boundaries, against the oracle's O9 sweep."""
    nsm = ns()
    s, z, y, a, delta, _ = sg.random_sweep_records(2000, seed + 300, n_delta=9)
    u = np.linspace(-4.0, 4.0, m).astype(np.float32)            # exactly m distinct candidates
    hit = np.random.default_rng(seed).random(len(z)) < 0.2
    z[hit] = np.random.default_rng(seed + 1).choice(u, int(hit.sum()))
    for fpl, fnl in ((0, 0), (250, 250), (400, 400)):   # infeasible, feasible, feasible
        T, best_o = O.sweep(s, z, y, a, delta, u, (3, 5, 7), fpl, fnl)
        best, code, _, _ = _gpu_sweep(nsm, s, z, y, a, delta, u, (3, 5, 7), fpl, fnl)
        assert (code == 7) == (not best_o["feasible"])
        for k_g, k_o in [("j", "j"), ("l", "l"), ("h", "h"), ("fp", "fp"), ("fn", "fn"),
                         ("uncertain", "U"), ("cost_ps", "cost")]:
            assert best[k_g] == best_o[k_o], (k_g, best, best_o)


@pytest.mark.parametrize("off,n", [(0, 4099), (1, 4099), (2, 100003), (3, 5), (1, 1), (0, 3)])
def test_sweep_hist_column_alignment(off, n):
    """Phase 1 reads 4 consecutive records per thread with 16-byte (s, z) and 4-byte
    (y, a) loads when every column is aligned, per-record loads otherwise and on the
    ragged end: record columns starting `off` records into their buffers (views, as a
    rank's unit slice of the flat record arrays) must give the oracle's tables."""
    nsm = ns()
    s, z, y, a, delta, u = sg.random_sweep_records(n + off, 900 + off, n_delta=9, m=8)
    dev = "cuda"
    T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).to(dev)
    sd, zd, yd, ad = T(s, np.float64), T(z, np.float32), T(y, np.uint8), T(a, np.uint8)
    dd, uu = T(delta, np.float64), T(u, np.float32)
    hist = torch.zeros(nsm.sweep_hist_words(len(delta), len(u)), dtype=torch.int64, device=dev)
    nsm.noscope_threshold_sweep(1, sd[off:], zd[off:], yd[off:], ad[off:], dd, uu, hist)
    nd, m = len(delta), len(u)
    tabs = {k: torch.zeros(nd * (m if k in ("FPf", "FNf", "GE", "GT") else 1), dtype=torch.int64,
                           device=dev) for k in ("F", "FPnf", "FNnf", "FPf", "FNf", "GE", "GT")}
    nsm.noscope_threshold_sweep(2, None, None, None, None, dd, uu, hist, (1, 10, 1000), 0, 0, tables=tabs)
    Tor = O.sweep_tables(s[off:], z[off:], y[off:], a[off:], delta, u)
    for k in ("F", "FPnf", "FNnf"):
        assert np.array_equal(tabs[k].cpu().numpy().astype(np.uint64), Tor[k]), k
    for k in ("FPf", "FNf", "GE", "GT"):
        assert np.array_equal(tabs[k].cpu().numpy().astype(np.uint64).reshape(nd, m), Tor[k]), k
