"""Multi-process parity on the real library: two ranks sharing
one B200 (gloo process group — the GPU box has one GPU, NCCL needs one GPU per
rank) run their units through noscope_cascade_run in chunks (dist.run_units), sum
their sweep histograms (C1) and gather labels to rank 0 (C2).  Labels and the
sweep's best triple must be identical to one process doing every unit, and the
labels must equal the oracle's per-unit cascade."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synthgen as sg
from gpu_util import requires_gpu

pytestmark = [pytest.mark.gpu, requires_gpu]

W, H, UNIT, N_UNITS, CHUNK, K = 160, 120, 300, 4, 128, 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_1703_02529_b200 import noscope as N
    arch_s = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch_s, 1)
    lr_w, lr_b = sg.lr_weights(10, 2)
    dd = N.DD(mode=1, metric=1, grid=10, t_diff_frames=K, delta_diff=-3.0,
              lr_weights=torch.from_numpy(lr_w).cuda(), lr_bias=float(lr_b))
    return N, dd, N.Arch(2, 32, 32), N.Weights(w), (arch_s, w, lr_w, lr_b)


def _scene(u):
    return sg.make_scene(sg.SceneSpec(W, H, UNIT, seed=40 + u, stream=u, prevalence=0.4))


def _shard(world, rank, lo, hi):
    from paper_1703_02529_b200 import dist as D
    from synthgen.gpu import GpuScene, truth_labeller_address
    N, dd, A, Wt, _ = _setup()
    lo_u, hi_u = D.unit_range(N_UNITS, world, rank)
    units = [dict(id=u, n_frames=UNIT, width=W, height=H) for u in range(lo_u, hi_u)]
    gs = {u["id"]: GpuScene(_scene(u["id"])) for u in units}
    buf = torch.empty((CHUNK, sg.frame_pitch(W, H)), dtype=torch.uint8, device="cuda")

    def make_frames(u, t0, m):
        return gs[u["id"]].render(buf, t0, m)[:m]

    rec = {}
    labels = D.run_units(N, units, make_frames, dd, A, Wt, lo, hi, truth_labeller_address(),
                         lambda u: gs[u["id"]].truth, chunk=CHUNK, device="cuda", records=rec)
    delta = torch.linspace(-3.0, 3.0, 9, dtype=torch.float64, device="cuda")
    u_c = torch.from_numpy(sg.logit_grid(12)).cuda()
    hist = torch.zeros(N.sweep_hist_words(9, 12), dtype=torch.int64, device="cuda")
    for u, s, z in zip(units, rec["scores"], rec["logits"]):
        a = N.noscope_sweep_records(s, gs[u["id"]].truth, 1, K, 1)
        N.noscope_threshold_sweep(1, s, z, gs[u["id"]].truth, a, delta, u_c, hist)
    D.allreduce_hist_(hist)
    best, _ = N.noscope_threshold_sweep(2, None, None, None, None, delta, u_c, hist, (1, 10, 1000), 60, 60)
    g = D.gather_labels_to_rank0(labels)
    return (None if g is None else g.cpu().numpy()), best, hist.cpu().numpy()


def _worker(rank, world, port, q, lo, hi):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, best, hist = _shard(world, rank, lo, hi)
        q.put((rank, None if g is None else g.tolist(), best, hist.tolist()))
    finally:
        dist.destroy_process_group()


def _oracle_units(lo, hi):
    _, _, _, _, (arch_s, w, lr_w, lr_b) = _setup()
    out = []
    for u in range(N_UNITS):
        sc = _scene(u)
        src = sg.render_frames(sc)[:, :W * H * 3].reshape(-1, H, W, 3)
        cfg = O.DDConfig(mode=1, metric=1, grid=10, t_diff_frames=K, delta_diff=-3.0, lr_w=lr_w, lr_b=lr_b)
        out.append(O.cascade(src, cfg, arch_s, w, lo, hi, sc.truth))
    return out


def test_two_ranks_equal_one_rank_and_oracle():
    # thresholds in gaps of the oracle's fired logits wider than the CNN parity bound
    z_all = np.sort(np.concatenate([r["logits"] for r in _oracle_units(-0.1, 0.1)]).astype(np.float64))
    gaps = np.diff(z_all)
    q = np.argsort(gaps)[::-1][:2]                     # the two widest gaps: NEG / UNC / POS all occur
    assert gaps[q].min() > 4e-2
    lo, hi = sorted(float(np.float32(0.5 * (z_all[i] + z_all[i + 1]))) for i in q)
    ref = _oracle_units(lo, hi)
    lab1, best1, hist1 = _shard(1, 0, lo, hi)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, lo, hi)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][1] == lab1.tolist() and res[1][1] is None
    assert res[0][2] == best1 and res[1][2] == best1
    assert res[0][3] == hist1.tolist() == res[1][3]
    for u in range(N_UNITS):                     # every unit's labels are the oracle cascade's
        assert np.array_equal(lab1[u * UNIT:(u + 1) * UNIT], ref[u]["labels"]), u


def test_flat_records_one_sweep_call_equals_per_unit_calls():
    """bench.py's config X builds one rank's sweep records back to back (run_units
    writing into flat buffers) and runs one record-builder + one phase-1 call: a
    unit's first K frames are forced fires (s = +inf), so the labels inherited
    across a unit boundary only reach the H1 row phase 2 never reads — the best
    triple equals the per-unit calls'."""
    from paper_1703_02529_b200 import dist as D
    from synthgen.gpu import GpuScene, truth_labeller_address
    N, dd, A, Wt, _ = _setup()
    lo, hi = -0.1, 0.1
    _, best_units, _ = _shard(1, 0, lo, hi)
    units = [dict(id=u, n_frames=UNIT, width=W, height=H) for u in range(N_UNITS)]
    gs = {u["id"]: GpuScene(_scene(u["id"])) for u in units}
    buf = torch.empty((CHUNK, sg.frame_pitch(W, H)), dtype=torch.uint8, device="cuda")
    s_all = torch.empty(N_UNITS * UNIT, dtype=torch.float64, device="cuda")
    z_all = torch.zeros(N_UNITS * UNIT, dtype=torch.float32, device="cuda")
    rec = {"flat": (s_all, z_all)}
    D.run_units(N, units, lambda u, t0, m: gs[u["id"]].render(buf, t0, m)[:m], dd, A, Wt, lo, hi,
                truth_labeller_address(), lambda u: gs[u["id"]].truth, chunk=CHUNK, device="cuda", records=rec)
    assert torch.isinf(s_all.view(N_UNITS, UNIT)[:, :K]).all()
    y_all = torch.cat([gs[u["id"]].truth[:UNIT] for u in units])
    a_all = N.noscope_sweep_records(s_all, y_all, 1, K, 1)
    delta = torch.linspace(-3.0, 3.0, 9, dtype=torch.float64, device="cuda")
    u_c = torch.from_numpy(sg.logit_grid(12)).cuda()
    hist = torch.zeros(N.sweep_hist_words(9, 12), dtype=torch.int64, device="cuda")
    N.noscope_threshold_sweep(1, s_all, z_all, y_all, a_all, delta, u_c, hist)
    best, _ = N.noscope_threshold_sweep(2, None, None, None, None, delta, u_c, hist, (1, 10, 1000), 60, 60)
    assert best == best_units
