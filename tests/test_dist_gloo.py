"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU driver's host
logic: unit sharding, the C1 histogram all-reduce (G-invariance of the sweep
counts) and the C2 label gather.  The histogram here is the sweep's definition
written out in the test (bins over candidates), evaluated with the oracle's
tables to show the summed histogram yields the single-process answer."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synthgen as sg
from paper_1703_02529_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _hist_np(s, z, y, a, delta, u):
    """H2[d][b][y], H1[d][a][y], checked, total — the sweep's record binning."""
    nd, m = len(delta), len(u)
    H2 = np.zeros((nd + 1, 2 * m + 1, 2), np.int64)
    H1 = np.zeros((nd + 1, 2, 2), np.int64)
    for i in range(len(s)):
        d = int(np.sum(delta < s[i]))
        b = int(np.sum(u < z[i]) + np.sum(u <= z[i]))
        H2[d, b, y[i]] += 1
        H1[d, a[i], y[i]] += 1
    return np.concatenate([H2.ravel(), H1.ravel(), [np.sum(s != -np.inf), len(s)]])


def _tables_from_hist(h, nd, m):
    B = 2 * m + 1
    H2 = h[:(nd + 1) * B * 2].reshape(nd + 1, B, 2)
    H1 = h[(nd + 1) * B * 2:(nd + 1) * B * 2 + (nd + 1) * 4].reshape(nd + 1, 2, 2)
    T = {"F": np.zeros(nd, np.uint64), "FPnf": np.zeros(nd, np.uint64), "FNnf": np.zeros(nd, np.uint64)}
    for k in ("FPf", "FNf", "GE", "GT"):
        T[k] = np.zeros((nd, m), np.uint64)
    for j in range(nd):
        fh = H2[j + 1:].sum(axis=0)                       # fired: d > j
        T["F"][j] = fh.sum()
        T["FPnf"][j] = H1[:j + 1, 1, 0].sum()
        T["FNnf"][j] = H1[:j + 1, 0, 1].sum()
        for t in range(m):
            T["FPf"][j, t] = fh[2 * t + 2:, 0].sum()
            T["GT"][j, t] = fh[2 * t + 2:].sum()
            T["GE"][j, t] = fh[2 * t + 1:].sum()
            T["FNf"][j, t] = fh[:2 * t + 1, 1].sum()
    T["checked"] = int(h[-2])
    T["total"] = int(h[-1])
    return T


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # sharding covers every unit exactly once, contiguous per rank
        lo, hi = D.unit_range(10, world, rank)
        # C1: sum of per-rank histograms of a split record set
        s, z, y, a, delta, u = sg.random_sweep_records(240, 5, n_delta=8, m=6)
        b = np.linspace(0, len(s), world + 1).astype(int)
        sl = slice(b[rank], b[rank + 1])
        h = torch.from_numpy(_hist_np(s[sl], z[sl], y[sl], a[sl], delta, u))
        D.allreduce_hist_(h)
        # C2: labels gathered in rank order
        lab = torch.full((3 + rank,), rank + 1, dtype=torch.uint8)
        g = D.gather_labels(lab, counts=[3 + r for r in range(world)])
        q.put((rank, (lo, hi), h.numpy().tolist(), g.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharding_allreduce_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [r[1] for r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == 10
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    s, z, y, a, delta, u = sg.random_sweep_records(240, 5, n_delta=8, m=6)
    full = _hist_np(s, z, y, a, delta, u)
    for r in res:                                   # identical, G-invariant sums on every rank
        assert np.array_equal(np.array(r[2]), full)
    T_h = _tables_from_hist(full, len(delta), len(u))
    T_o = O.sweep_tables(s, z, y, a, delta, u)
    for k in ("F", "FPnf", "FNnf", "FPf", "FNf", "GE", "GT"):
        assert np.array_equal(T_h[k], T_o[k]), k
    b_h = O.sweep_best(T_h, (1, 10, 1000), 4, 4)
    b_o = O.sweep_best(T_o, (1, 10, 1000), 4, 4)
    assert b_h == b_o
    g = res[0][3]
    assert g == [1, 1, 1, 2, 2, 2, 2]


def test_unit_range_partition():
    for U in (1, 7, 8, 192):
        for G in (1, 2, 4, 8):
            seen = []
            for r in range(G):
                lo, hi = D.unit_range(U, G, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(U))


# ---------------------------------------------------------------- run_units + C1 + C2
class _StubNS:
    """CPU stand-in with the binding's call signatures (test-only).  Its 'cascade'
    carries state across chunks (label_t = (bytes_t + carry) mod 3 mod 2), so the
    result depends on the chunk loop carrying state within a unit and resetting
    it between units — the logic run_units owns."""

    def noscope_stream_state_init(self, dd):
        return torch.zeros(1, dtype=torch.int64)

    def noscope_cascade_run(self, dd, arch, w, lo, hi, frames, W, H, state, labeller, user, seg_offset=0,
                            frame_index_base=0, ws=None, labels=None, scores_out=None, logits_out=None):
        v = frames.to(torch.int64).sum(dim=1)
        for i in range(len(v)):
            state[0] = (v[i] + state[0]) % 3
            labels[i] = int(state[0] % 2)
        if scores_out is not None:
            scores_out.copy_((v % 11).double())
        if logits_out is not None:
            logits_out.copy_((v % 7).float() - 3.0)


N_UNITS, UNIT_LEN, CHUNK = 6, 23, 5


def _units():
    return [dict(id=i, n_frames=UNIT_LEN, width=4, height=4) for i in range(N_UNITS)]


def _make_frames(u, t0, m):
    rng = np.random.default_rng(1000 * u["id"] + 7)
    f = rng.integers(0, 256, (UNIT_LEN, 16), dtype=np.uint8)
    return torch.from_numpy(f[t0:t0 + m].copy())


def _truth(u):
    return (np.random.default_rng(u["id"]).random(UNIT_LEN) < 0.4).astype(np.uint8)


def _shard_run(world, rank):
    """This rank's units -> (labels, per-record histogram over the unit records)."""
    lo_u, hi_u = D.unit_range(N_UNITS, world, rank)
    units = _units()[lo_u:hi_u]
    rec = {}
    lab = D.run_units(_StubNS(), units, _make_frames, None, None, None, 0.0, 0.0, 0, lambda u: 0,
                      chunk=CHUNK, device="cpu", records=rec)
    delta, u = np.array([1.5, 4.5, 8.5]), np.float32([-2.5, 0.0, 2.0])

    def hist_fn(h):
        for uu, s, z in zip(units, rec["scores"], rec["logits"]):
            y = _truth(uu)
            a = O.build_records(s.numpy(), y, 1, 2)
            h += torch.from_numpy(_hist_np(s.numpy(), z.numpy(), y, a, delta, u))

    def eval_fn(h):
        T = _tables_from_hist(h.numpy(), len(delta), len(u))
        return O.sweep_best(T, (1, 10, 1000), 10, 10)

    n_words = (len(delta) + 1) * (2 * len(u) + 1) * 2 + (len(delta) + 1) * 4 + 2
    best, _ = D.distributed_sweep(hist_fn, eval_fn, n_words, "cpu")
    return lab, best


def _worker_units(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lab, best = _shard_run(world, rank)
        g = D.gather_labels_to_rank0(lab)
        q.put((rank, None if g is None else g.numpy().tolist(), best))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_run_units_and_distributed_sweep_are_world_size_invariant(world):
    """labels (gathered to rank 0) and the sweep's best triple
    (C1 all-reduce of the local histograms) are identical for G = 1 and G = world."""
    lab1, best1 = _shard_run(1, 0)                       # single process, no process group
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_units, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == lab1.numpy().tolist()            # rank 0 holds every unit's labels in order
    assert all(r[1] is None for r in res[1:])            # a gather, not an all-gather
    assert all(r[2] == best1 for r in res)               # every rank evaluates the same summed counts
    # the stub's state carry matters: chunking without carry would change labels
    assert len(lab1) == N_UNITS * UNIT_LEN
