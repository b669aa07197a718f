#!/usr/bin/env python
"""Benchmark of the NoScope cascade hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the metric's config): one hour of a
synthetic fixed-angle 640x480 webcam at 30 fps = 108,000 frames (99.5 GB,
resident in HBM before the timed region), blocked-MSE difference detector
(10x10 grid, LR weights ~U[0,1], bias -4) against frame t-30, t_skip = 1,
delta_diff at the 85th percentile of the unit's scores, specialized CNN
L2/C32/D32 (random He-normal bf16 weights), c_low/c_high at the 30%/70%
logit quantiles of fired frames, ground-truth stand-in labeller.
One step = noscope_cascade_run over the whole unit (state re-initialised).
Inputs (99.5 GB) exceed L2 (126 MB), so no L2 flush is needed between steps.

Multi-GPU (torchrun, one process per GPU): every rank processes its own
stream's hour (weak scaling); labels are gathered to rank 0 over NCCL inside
the timed region; time = max over ranks of device-event time.

--impl reference: the CPU oracle (oracle/) on a bounded sample of the same
workload, on this host's cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# streaming-read ceilings of this part, measured by tools/read_bw.cu (grid-stride uint4
# loads) and tools/bulk_ring_bw.cu (dd_kernel's band ring with no compute), GB/s
READ_CEIL_LDG = 6970.3
READ_CEIL_BULK = 7534.6
sys.path.insert(0, ROOT)

W_SRC, H_SRC, OUT = 640, 480, 50
UNIT = 108_000
K_LAG = 30
GRID = 10
ARCH = (2, 32, 32)
CONFIG_NAME = "webcam-1h: 108k 640x480 frames, blocked-MSE (10x10, LR) vs t-30, t_skip=1, CNN L2C32D32"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--frames", type=int, default=UNIT, help="frames per unit (default 1 h)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-extras", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-frames", type=int, default=192)
    p.add_argument("--e2e-frames", type=int, default=13500)
    p.add_argument("--workload", default="webcam", choices=["webcam", "x"],
                   help="webcam: BASELINE configs[1] (the metric's config); x: configs[4], "
                        "8 streams x 24 h sharded over the ranks")
    p.add_argument("--x-streams", type=int, default=8)
    p.add_argument("--x-hours", type=int, default=24)
    return p.parse_args()


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def maybe_self_launch(args):
    """`--gpus N` outside torchrun: re-launch this script as N ranks (one process per
    GPU) under torch.distributed.run on this node; fails if fewer than N GPUs."""
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            sys.exit(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}")
        return
    if args.gpus <= 1:
        return
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, {have} visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


class _StdoutToStderr:
    """fd 1 -> stderr while NCCL creates / destroys communicators (it logs to stdout)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def destroy_dist():
    import torch.distributed as dist
    if dist.is_initialized():
        with _StdoutToStderr():
            dist.destroy_process_group()


def init_dist(world, device):
    """One process per GPU over NCCL (NCCL_DEBUG=INFO so the init lines show nranks)."""
    import torch.distributed as dist
    if world > 1 or "WORLD_SIZE" in os.environ:   # under torchrun: NCCL even for one rank
        import torch
        # torch pre-sets NCCL_DEBUG=VERSION; INFO (init subsystem) so the log shows nranks
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("", "VERSION", "WARN"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        # NCCL prints its banner and logs to stdout: create the communicator (one warm-up
        # all-reduce) with fd 1 pointed at stderr, so stdout carries only the JSON line
        with _StdoutToStderr():
            dist.init_process_group("nccl", device_id=device)
            t = torch.ones(1, device=device)
            dist.all_reduce(t)
            torch.cuda.synchronize()


# cost-model timings for the in-step sweep (ps per frame): T_MSE and T_SNN as measured
# on B200 in round 1 (dd_kernel 14.66 ms / 108k frames; CNN 0.86 ms / 16.2k fired
# frames), T_full = the paper's YOLOv2 at 80 fps on a P100
SWEEP_TIMING = (135_726, 53_050, 12_500_000_000)
SWEEP_M = 100


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- workload
def make_weights():
    import synthgen as sg
    arch = sg.CnnArch(*ARCH)
    return arch, sg.he_normal_weights(arch, 3), sg.lr_weights(GRID, 3)


def setup_gpu(rank, n_frames, device):
    """Render the unit on the device (decode stand-in) and pick thresholds."""
    import torch
    import synthgen as sg
    from paper_1703_02529_b200 import noscope as N
    from synthgen.gpu import GpuScene

    sc = sg.make_scene(sg.SceneSpec(W_SRC, H_SRC, n_frames, seed=2, stream=rank))
    gs = GpuScene(sc, device=device)
    pitch = sg.frame_pitch(W_SRC, H_SRC)
    frames = torch.empty((n_frames, pitch), dtype=torch.uint8, device=device)
    step = 4096
    for t0 in range(0, n_frames, step):
        gs.render(frames[t0:t0 + step], t0, min(step, n_frames - t0))
    arch_s, w, (lr_w, lr_b) = make_weights()
    dd = N.DD(mode=1, metric=1, out_w=OUT, out_h=OUT, grid=GRID, t_diff_frames=K_LAG, t_skip_frames=1,
              delta_diff=0.0, lr_weights=torch.from_numpy(lr_w).to(device), lr_bias=float(lr_b))
    # delta_diff = 85th percentile of the unit's finite scores
    state = N.noscope_stream_state_init(dd)
    probe = N.noscope_diff_detect(dd, frames, W_SRC, H_SRC, state=state, compact=False)
    sc_t = probe["score"]
    fin = sc_t[torch.isfinite(sc_t)]
    dd.delta_diff = float(torch.quantile(fin[:: max(1, fin.numel() // 100000)].float(), 0.85).item())
    del probe
    arch = N.Arch(*ARCH)
    W = N.Weights(w, device=device)
    state = N.noscope_stream_state_init(dd)
    det = N.noscope_diff_detect(dd, frames, W_SRC, H_SRC, state=state)
    nf = int(det["n_fired"].item())
    z = N.noscope_specialized_infer(arch, W, det["small"], idx=det["idx"][:nf])
    lo = float(torch.quantile(z.float(), 0.3).item())
    hi = float(torch.quantile(z.float(), 0.7).item())
    del det, z
    torch.cuda.empty_cache()
    return dict(scene=sc, gs=gs, frames=frames, dd=dd, arch=arch, W=W, lo=lo, hi=hi, w=w,
                lr=(lr_w, lr_b), pitch=pitch)


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1703_02529_b200 import noscope as N
    from synthgen.gpu import truth_labeller_address

    from paper_1703_02529_b200 import dist as D
    import synthgen as sg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    init_dist(world, device)   # one process per GPU; the NCCL communicator bound to this rank's device
    n = args.frames
    S = setup_gpu(rank, n, device)
    dd, arch, W = S["dd"], S["arch"], S["W"]
    ws = N.workspace(N.OP_CASCADE_RUN, dd, arch, n, device=device)
    state = torch.empty(max(1, N.lib().noscope_stream_state_bytes(__import__("ctypes").byref(dd.c()))),
                        dtype=torch.uint8, device=device)
    labels = torch.empty(n, dtype=torch.uint8, device=device)
    gathered = torch.empty(n * world, dtype=torch.uint8, device=device) if rank == 0 else None
    lab_fn = truth_labeller_address()
    stream = torch.cuda.current_stream()
    stats = {}
    # CBO sweep records of the step: s = DD score, z = CNN logit (written for
    # fired frames; delta candidates are >= the cascade's delta, so every frame fired
    # under a candidate was fired in the step and has its logit), y = reference label
    # (stand-in labeller = ground truth), a = label emitted when not fired
    scores = torch.empty(n, dtype=torch.float64, device=device)
    logits = torch.zeros(n, dtype=torch.float32, device=device)
    a_rec = torch.empty(n, dtype=torch.uint8, device=device)
    truth = S["gs"].truth
    ul = torch.from_numpy(sg.logit_grid(SWEEP_M)).to(device)
    hist = torch.zeros(N.sweep_hist_words(SWEEP_M, SWEEP_M), dtype=torch.int64, device=device)
    sws = N.workspace(N.OP_THRESHOLD_SWEEP, None, None, 0, SWEEP_M, SWEEP_M, device=device)
    fp_lim = fn_lim = (n * world) // 100                     # FP* = FN* = 1%
    sweep = {"dl": None, "best": N.pinned_sweep_best()}     # phase 2 result: async copy, no host sync

    def step(stage_acc=None):
        N.lib().noscope_stream_state_init(__import__("ctypes").byref(dd.c()), N._ptr(state), N._stream())
        stage = [] if stage_acc is not None else None
        out = N.noscope_cascade_run(dd, arch, W, S["lo"], S["hi"], S["frames"], W_SRC, H_SRC, state,
                                    lab_fn, truth, ws=ws, labels=labels, logits_out=logits, scores_out=scores,
                                    want_stats=not stats, stage_ms=stage)
        if "stats" in out:
            stats.update(out["stats"])
        if stage_acc is not None:
            stage_acc.append(stage)
        if sweep["dl"] is None:    # candidates from the first (warm-up) step: 100 quantiles of s >= delta
            fired_s = scores[scores > dd.delta_diff]
            q = torch.quantile(fired_s[:: max(1, fired_s.numel() // 100000)], torch.linspace(
                0, 1, SWEEP_M - 1, dtype=torch.float64, device=device))
            grid = torch.unique(torch.cat([torch.tensor([dd.delta_diff], dtype=torch.float64, device=device), q]))
            sweep["dl"] = grid[:SWEEP_M].contiguous()
        dl = sweep["dl"]
        N.noscope_sweep_records(scores, truth, 1, K_LAG, 1, a_out=a_rec)
        hist.zero_()
        N.noscope_threshold_sweep(1, scores, logits, truth, a_rec, dl, ul, hist)
        D.allreduce_hist_(hist)                                                   # C1 (NCCL)
        N.noscope_threshold_sweep(2, None, None, None, None, dl, ul, hist, SWEEP_TIMING, fp_lim, fn_lim, ws=sws,
                                  best_out=sweep["best"])
        D.gather_labels_to_rank0(labels, out=gathered)                            # C2 (NCCL gather)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    stage_acc = []
    l0 = N.launch_count()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(stage_acc)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = N.launch_count() - l0 + args.steps      # + the stand-in labeller kernel per step
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    per_rank = [ms]
    if dist.is_initialized():
        t = torch.zeros(world, device=device)
        t[rank] = ms
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        per_rank = [float(v) for v in t.tolist()]
    ms = max(per_rank)
    ms_step = ms / args.steps
    fps = n * world / (ms_step / 1e3)
    stage = np.mean(np.array(stage_acc), axis=0)   # 7 stages, ms

    hbm, bf16, bf16_sus, peak_kind = measured_peaks()
    # dominant kernel: dd_kernel (fused downsample + DD score); algorithmic bytes per launch =
    # frames downsampled x (source frame read + small frame write)
    ds_bytes = n * (W_SRC * H_SRC * 3 + OUT * OUT * 3)
    ds_ms = float(stage[0])
    achieved = ds_bytes / (ds_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_dd_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    nf = stats.get("n_fired", 0)
    cnn_flops = nf * cnn_flops_per_frame(ARCH)
    line = {
        "metric": "cascade frames/sec (diff+CNN+routing)",
        "value": round(fps, 1),
        "unit": "frames/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8/int64/f64 (DD), bf16->f32 (CNN)",
        "data": "synthetic fixed-angle webcam (static textured background, sensor noise, moving "
                "rectangles), random-init He-normal CNN weights; generated on device before timing",
        "config": {"workload": CONFIG_NAME, "frames_per_gpu": n, "source": f"{W_SRC}x{H_SRC}x3 u8",
                   "dd": "mode 1 (t-30), blocked 10x10 + LR, t_skip 1",
                   "delta_diff": dd.delta_diff, "c_low_logit": S["lo"], "c_high_logit": S["hi"],
                   "cnn": "L2C32D32", "l2_flush": "not needed: 99.5 GB input per GPU > 126 MB L2",
                   "parallelism": f"dp{world} (units sharded by stream)"},
        "roofline": {"bound": "hbm", "kernel": "dd_kernel", "achieved": round(achieved, 1),
                     "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "peak_source": peak_kind, "traffic": traffic,
                     "algorithmic_bytes_per_launch": ds_bytes, "avg_launch_ms": round(ds_ms, 4),
                     # dd_kernel's traffic is >99% reads; the copy peak above counts read+write.
                     # Streaming-read ceilings measured on B200 (profiles/r01/read_ceiling.txt):
                     "read_ceilings_GBps": {"ldg_stream": READ_CEIL_LDG, "bulk_ring": READ_CEIL_BULK},
                     "frac_of_bulk_ring_ceiling": round(achieved / READ_CEIL_BULK, 4)},
        "stage_ms": {k: round(float(v), 4) for k, v in zip(
            ["dd_kernel", "dd_tail", "compaction", "cnn", "routing", "labeller",
             "labels_state"], stage)},
        "run_stats": stats,
        "per_rank": [{"rank": r, "ms_per_step": round(v / args.steps, 4),
                      "fps": round(n / (v / args.steps / 1e3), 1)} for r, v in enumerate(per_rank)],
        "step": "noscope_cascade_run over the unit (downsample, DD, compaction, CNN, routing, stand-in "
                "labeller, labels) + sweep records + noscope_threshold_sweep phase 1 + C1 all_reduce of "
                "the sweep histogram + phase 2 (best triple to host) + C2 gather of the labels to rank 0",
        "sweep": {k: N.sweep_best_dict(sweep["best"])[k] for k in ("j", "l", "h", "feasible", "cost_ps", "fp", "fn",
                                                                    "fired", "uncertain", "checked", "total")},
        "cnn": {"frames": nf, "tflops": round(cnn_flops / (stage[3] / 1e3) / 1e12, 2) if stage[3] > 0 else None},
        "gpu_launches": int(launches),
    }
    if rank == 0:
        with ClockSampler(local) as _:
            pass
        line["clocks"] = clk.summary()
    if not args.no_e2e:
        line["e2e"] = run_e2e(args, S, device, world)
    if not args.no_extras and rank == 0:
        line["tskip15"] = run_tskip(S, device, 15)
    del S["frames"]
    torch.cuda.empty_cache()
    if not args.no_extras and rank == 0:
        # measured per-frame costs (ps) for the CBO cost model: T_MSE from the DD
        # kernel, T_SNN from the cascade's CNN stage; T_full = the paper's YOLOv2
        # (80 fps on a P100, P:162-164 — the reference NN is not run here)
        t_mse = int(stage[0] * 1e9 / n) if stage[0] > 0 else 1000
        t_snn = int(stage[3] * 1e9 / max(nf, 1)) if stage[3] > 0 else 20000
        line["extras"] = run_extras(device, (t_mse, t_snn, 12_500_000_000))
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args, S)
    if rank == 0:
        print(json.dumps(line), flush=True)
    destroy_dist()


def run_x(args):
    """BASELINE configs[4]: S streams x H hours of 640x480 webcam at
    30 fps, units = (stream, hour) of 108,000 frames (R-19), unit u on rank
    floor(u*G/U).  Frames are rendered on device in chunks of 27,000 (the decode
    stand-in, untimed); each chunk goes through noscope_cascade_run with the unit's
    carried state; the timed work per rank = the sum of its cascade intervals (CUDA
    events) + the C1 sweep (phase 1 over every unit's records, all_reduce, phase 2)
    + the C2 label gather to rank 0; value = all frames / max over ranks."""
    import ctypes
    import torch
    import torch.distributed as dist
    import synthgen as sg
    from paper_1703_02529_b200 import dist as D
    from paper_1703_02529_b200 import noscope as N
    from synthgen.gpu import GpuScene, truth_labeller_address

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    init_dist(world, device)
    unit_len = args.frames
    units = [dict(stream=st, hour=h, n_frames=unit_len, width=W_SRC, height=H_SRC)
             for st in range(args.x_streams) for h in range(args.x_hours)]
    lo_u, hi_u = D.unit_range(len(units), world, rank)
    mine = units[lo_u:hi_u]
    scenes = {}
    for u in mine:
        if u["stream"] not in scenes:   # seed 100 + stream; one scene per 24 h stream
            sc = sg.make_scene(sg.SceneSpec(W_SRC, H_SRC, args.x_hours * unit_len, seed=100 + u["stream"],
                                            stream=u["stream"]))
            scenes[u["stream"]] = GpuScene(sc, device=device)
    chunk = 27_000          # 4 chunks per one-hour unit (24.9 GB of frames per chunk)
    pitch = sg.frame_pitch(W_SRC, H_SRC)
    buf = torch.empty((chunk, pitch), dtype=torch.uint8, device=device)

    def make_frames(u, t0, m):
        scenes[u["stream"]].render(buf, u["hour"] * unit_len + t0, m)
        return buf[:m]

    arch_s, w, (lr_w, lr_b) = make_weights()
    # the W configuration's thresholds, fixed for every unit (delta at the 85th percentile of
    # a unit's scores and c_low / c_high at the 30 / 70 % fired-logit quantiles of stream 0, hour 0)
    S = setup_gpu(0, min(unit_len, 16384), device)
    dd, arch, Wt, lo, hi = S["dd"], S["arch"], S["W"], S["lo"], S["hi"]
    del S
    torch.cuda.empty_cache()
    ws = N.workspace(N.OP_CASCADE_RUN, dd, arch, chunk, device=device)
    truth_of = lambda u: scenes[u["stream"]].truth[u["hour"] * unit_len:(u["hour"] + 1) * unit_len]
    lab_fn = truth_labeller_address()
    # warm-up: one chunk (its scores also fix the sweep's delta candidates: 100
    # quantiles of the fired scores, as in the webcam line)
    rec0 = {}
    D.run_units(N, [dict(mine[0], n_frames=chunk)], make_frames, dd, arch, Wt, lo, hi, lab_fn, truth_of,
                chunk=chunk, ws=ws, device=device, records=rec0)
    s0 = rec0["scores"][0]
    fired_s = s0[s0 > dd.delta_diff]
    q = torch.quantile(fired_s, torch.linspace(0, 1, SWEEP_M - 1, dtype=torch.float64, device=device))
    dl = torch.unique(torch.cat([torch.tensor([dd.delta_diff], dtype=torch.float64, device=device), q]))
    ul = torch.from_numpy(sg.logit_grid(SWEEP_M)).to(device)
    hist = torch.zeros(N.sweep_hist_words(dl.numel(), SWEEP_M), dtype=torch.int64, device=device)
    sws = N.workspace(N.OP_THRESHOLD_SWEEP, None, None, 0, dl.numel(), SWEEP_M, device=device)
    best = N.pinned_sweep_best()
    total = len(units) * unit_len
    gathered = torch.empty(total, dtype=torch.uint8, device=device) if rank == 0 else None
    # this rank's records, all units back to back: one record-builder and one phase-1 call
    # cover every unit (a unit's first K_LAG frames are forced fires, s = +inf, fired for
    # every delta candidate, so the label they would inherit across the unit boundary only
    # lands in the H1 row d = n_delta, which phase 2 never reads: every count the sweep
    # reads, and so the best triple, equals the per-unit calls)
    n_mine = sum(u["n_frames"] for u in mine)
    s_all = torch.empty(n_mine, dtype=torch.float64, device=device)
    z_all = torch.zeros(n_mine, dtype=torch.float32, device=device)
    y_all = torch.cat([truth_of(u) for u in mine]) if mine else torch.empty(0, dtype=torch.uint8, device=device)
    a_all = torch.empty(max(n_mine, 1), dtype=torch.uint8, device=device)
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    timer, rec = [], {"flat": (s_all, z_all)}
    with ClockSampler(local) as clk:
        labels = D.run_units(N, mine, make_frames, dd, arch, Wt, lo, hi, lab_fn, truth_of, chunk=chunk, ws=ws,
                             device=device, timer=timer, records=rec)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if n_mine:
            N.noscope_sweep_records(s_all, y_all, 1, K_LAG, 1, a_out=a_all[:n_mine])
            N.noscope_threshold_sweep(1, s_all, z_all, y_all, a_all[:n_mine], dl, ul, hist)
        D.allreduce_hist_(hist)                                                            # C1
        N.noscope_threshold_sweep(2, None, None, None, None, dl, ul, hist, SWEEP_TIMING, total // 100,
                                  total // 100, ws=sws, best_out=best)
        D.gather_labels_to_rank0(labels, out=gathered)                                     # C2
        e1.record()
        torch.cuda.synchronize()
    best = N.sweep_best_dict(best)
    cascade_ms = sum(a.elapsed_time(b) for a, b in timer)
    ms = cascade_ms + e0.elapsed_time(e1)
    per_rank = [ms]
    if dist.is_initialized():
        t = torch.zeros(world, device=device)
        t[rank] = ms
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        per_rank = [float(v) for v in t.tolist()]
    tmax = max(per_rank)
    if rank == 0:
        line = {"metric": "cascade frames/sec (diff+CNN+routing)", "value": round(total / (tmax / 1e3), 1),
                "unit": "frames/s", "n_gpus": world, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u8/int64/f64 (DD), bf16->f32 (CNN)",
                "data": "synthetic fixed-angle webcam streams rendered on device in 27,000-frame chunks "
                        "(untimed), random-init CNN weights",
                "config": {"workload": f"x: {args.x_streams} streams x {args.x_hours} h at 30 fps, 640x480, "
                                       f"units of {unit_len} frames sharded over {world} GPU(s)",
                           "frames_total": total, "units": len(units), "chunk": chunk,
                           "dd": "mode 1 (t-30), blocked 10x10 + LR, t_skip 1", "cnn": "L2C32D32",
                           "parallelism": f"dp{world} (units by stream and hour)"},
                "ms_total": round(tmax, 2), "cascade_ms_rank0": round(cascade_ms, 2),
                "per_rank_ms": [round(v, 2) for v in per_rank],
                "sweep": {k: best[k] for k in ("j", "l", "h", "feasible", "cost_ps", "fp", "fn", "uncertain")},
                "labels_positive_frac": round(float(gathered.float().mean().item()), 4) if gathered is not None
                else None,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    destroy_dist()


def run_tskip(S, device, t_skip, steps=5):
    """The same webcam hour with the paper's frame skipping ("every 15
    frames"): only frames with tau mod t_skip == 0 are read and scored (their t-30
    anchors are checked frames too), skipped frames inherit the last checked label.
    Same thresholds; device-timed like the main line, whole cascade per step."""
    import copy
    import ctypes
    import torch
    from paper_1703_02529_b200 import noscope as N
    from synthgen.gpu import truth_labeller_address
    dd = copy.copy(S["dd"])
    dd.t_skip_frames = t_skip
    n = S["frames"].shape[0]
    ws = N.workspace(N.OP_CASCADE_RUN, dd, S["arch"], n, device=device)
    state = torch.empty(max(1, N.lib().noscope_stream_state_bytes(ctypes.byref(dd.c()))), dtype=torch.uint8,
                        device=device)
    labels = torch.empty(n, dtype=torch.uint8, device=device)
    lab_fn = truth_labeller_address()
    stats = {}

    def step():
        N.lib().noscope_stream_state_init(ctypes.byref(dd.c()), N._ptr(state), N._stream())
        out = N.noscope_cascade_run(dd, S["arch"], S["W"], S["lo"], S["hi"], S["frames"], W_SRC, H_SRC, state,
                                    lab_fn, S["gs"].truth, ws=ws, labels=labels, want_stats=not stats)
        if "stats" in out:
            stats.update(out["stats"])

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    checked = n - stats.get("n_skipped", 0)
    src = checked * (W_SRC * H_SRC * 3 + OUT * OUT * 3)
    return {"t_skip": t_skip, "frames": n, "checked": checked, "ms_per_step": round(ms, 4),
            "fps": round(n / (ms / 1e3), 1), "checked_source_GBps": round(src / ms / 1e6, 1),
            "run_stats": stats}


def cnn_flops_per_frame(arch):
    L, Cb, D = arch
    h, cin, f = 50, 3, 0
    for l in range(L):
        cout = Cb * 2 ** l
        f += 2 * h * h * 9 * cin * cout
        h //= 2
        cin = cout
    K = h * h * cin
    return f + 2 * K * D + 2 * D


def run_e2e(args, S, device, world):
    """Same metric through the public C ABI with HOST buffers: each step copies
    the unit's frames from pinned host memory (H2D) chunk by chunk, runs the
    cascade on each chunk with carried stream state, and reads the labels back
    (D2H), on two streams so copies overlap compute.  Bounded unit size."""
    import torch
    from paper_1703_02529_b200 import noscope as N
    from synthgen.gpu import truth_labeller_address
    n = min(args.e2e_frames, args.frames)
    chunk = 1024
    pitch = S["pitch"]
    host = torch.empty((n, pitch), dtype=torch.uint8, pin_memory=True)
    host.copy_(S["frames"][:n], non_blocking=False)
    lab_host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dev_buf = [torch.empty((chunk, pitch), dtype=torch.uint8, device=device) for _ in range(2)]
    labels = torch.empty(n, dtype=torch.uint8, device=device)
    dd, arch, W = S["dd"], S["arch"], S["W"]
    ws = N.workspace(N.OP_CASCADE_RUN, dd, arch, chunk, device=device)
    import ctypes
    state = torch.empty(max(1, N.lib().noscope_stream_state_bytes(ctypes.byref(dd.c()))), dtype=torch.uint8,
                        device=device)
    copy_s = torch.cuda.Stream(device=device)
    comp_s = torch.cuda.current_stream()
    lab_fn = truth_labeller_address()

    def step():
        N.lib().noscope_stream_state_init(ctypes.byref(dd.c()), N._ptr(state), N._stream(comp_s))
        done = [torch.cuda.Event() for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        for c, t0 in enumerate(range(0, n, chunk)):
            b = c & 1
            m = min(chunk, n - t0)
            with torch.cuda.stream(copy_s):
                if c >= 2:
                    copy_s.wait_event(done[b])
                dev_buf[b][:m].copy_(host[t0:t0 + m], non_blocking=True)
                ready[b].record(copy_s)
            comp_s.wait_event(ready[b])
            N.noscope_cascade_run(dd, arch, W, S["lo"], S["hi"], dev_buf[b][:m], W_SRC, H_SRC, state,
                                  lab_fn, S["gs"].truth, seg_offset=t0, frame_index_base=t0, ws=ws,
                                  labels=labels[t0:t0 + m], stream=comp_s)
            done[b].record(comp_s)
        lab_host.copy_(labels, non_blocking=True)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    steps = max(2, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp_s)
    for _ in range(steps):
        step()
    e1.record(comp_s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del host
    peak = pinned_h2d_peak(device)
    h2d = n * pitch / ms / 1e6
    return {"value": round(n * world / (ms / 1e3), 1), "unit": "frames/s",
            "h2d_bytes_per_step": n * pitch, "d2h_bytes_per_step": n,
            "frames_per_step": n, "chunk": chunk, "ms_per_step": round(ms, 3),
            "h2d_GBps": round(h2d, 1), "pinned_h2d_peak_GBps": peak,
            "frac_of_h2d_peak": round(h2d / peak, 4) if peak else None}


def pinned_h2d_peak(device, nbytes=1 << 30, reps=5):
    """Measured pinned host -> device copy bandwidth (GB/s, best of reps, CUDA events):
    the ceiling of the e2e path, whose input crosses PCIe / C2C every step."""
    import torch
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(nbytes, dtype=torch.uint8, device=device)
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.copy_(host, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / e0.elapsed_time(e1) / 1e6)
    del host, dev
    return round(best, 1)


def run_extras(device, timing=(1000, 20000, 12_500_000_000)):
    """Secondary measurements of the other BASELINE configs (not the headline)."""
    import torch
    import synthgen as sg
    from paper_1703_02529_b200 import noscope as N
    out = {}
    _, bf16, bf16_sus, _ = measured_peaks()
    # configs[2]: CNN grid, 65,536 frames per arch
    nG = 65536
    sc = sg.make_scene(sg.SceneSpec(50, 50, nG, seed=3, prevalence=0.15))
    gs = __import__("synthgen.gpu", fromlist=["GpuScene"]).GpuScene(sc, device=device)
    small = torch.empty((nG, 7504), dtype=torch.uint8, device=device)
    gs.render(small, 0, nG)
    grid = {}
    for a in sg.ARCH_GRID:
        w = sg.he_normal_weights(a, 3)
        A, Wt = N.Arch(a.n_conv, a.base_filters, a.dense), N.Weights(w, device=device)
        ws = N.workspace(N.OP_SPECIALIZED_INFER, None, A, nG, device=device)
        logits = torch.empty(nG, dtype=torch.float32, device=device)
        for _ in range(2):
            N.noscope_specialized_infer(A, Wt, small, ws=ws, logits=logits)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            N.noscope_specialized_infer(A, Wt, small, ws=ws, logits=logits)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        fl = cnn_flops_per_frame((a.n_conv, a.base_filters, a.dense)) * nG
        grid[a.name] = {"ms": round(ms, 3), "fps": round(nG / ms * 1e3, 1),
                        "tflops": round(fl / ms / 1e9, 1), "frac_of_bf16_peak": round(fl / ms / 1e9 / bf16, 4)}
        del ws
    # ncu tensor-pipe activity of the same calls (captured once per kernel change by
    # tools/gpu_cnn_tensor.sh; a profiler cannot run inside the timed bench)
    tpath = os.path.join(ROOT, "profiles", "r02", "cnn_tensor_pipe.json")
    if os.path.exists(tpath):
        tp = json.load(open(tpath))["archs"]
        for name, rec in grid.items():
            if name in tp:
                rec["ncu_tensor_pipe_active_pct"] = tp[name]["tensor_pipe_active_pct"]
    out["cnn_grid_65536"] = grid
    # the paper's remaining search configurations (C = 16 and D = 64 / 256)
    extra = {}
    for a in sg.PAPER_GRID:
        if a.name in grid:
            continue
        w = sg.he_normal_weights(a, 3)
        A, Wt = N.Arch(a.n_conv, a.base_filters, a.dense), N.Weights(w, device=device)
        ws = N.workspace(N.OP_SPECIALIZED_INFER, None, A, nG, device=device)
        logits = torch.empty(nG, dtype=torch.float32, device=device)
        ms = _time_ms(lambda: N.noscope_specialized_infer(A, Wt, small, ws=ws, logits=logits))
        fl = cnn_flops_per_frame((a.n_conv, a.base_filters, a.dense)) * nG
        extra[a.name] = {"ms": round(ms, 3), "fps": round(nG / ms * 1e3, 1), "tflops": round(fl / ms / 1e9, 1),
                         "frac_of_bf16_peak": round(fl / ms / 1e9 / bf16, 4)}
        del ws
    out["cnn_paper_grid_rest_65536"] = extra
    out["tiny_T"] = tiny_config(device)
    out["next_rows"] = next_rows_extras(device, sc, gs, small, nG)
    # configs[3]: sweep over 1M labelled records, 100 x 100 candidates
    rng = np.random.default_rng(4)
    M = 1_000_000
    y = (rng.random(M) < 0.15).astype(np.uint8)
    s = np.where(rng.random(M) < 0.05, -np.inf, rng.gamma(2.0, 10.0, M) + 40.0 * y)
    z = (rng.normal(0, 1, M) + 2.5 * y - 1.0).astype(np.float32)
    a_ = np.where(np.isinf(s), y, 0).astype(np.uint8)
    T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).to(device)
    sd, zd, yd, ad = T(s, np.float64), T(z, np.float32), T(y, np.uint8), T(a_, np.uint8)
    dl, ul = T(sg.delta_grid(s, 100), np.float64), T(sg.logit_grid(100), np.float32)
    hist = torch.zeros(N.sweep_hist_words(100, 100), dtype=torch.int64, device=device)
    ws = N.workspace(N.OP_THRESHOLD_SWEEP, None, None, 0, 100, 100, device=device)
    # (timing: B200-measured T_MSE / T_SNN in ps, see the caller)
    for _ in range(2):
        hist.zero_()
        N.noscope_threshold_sweep(3, sd, zd, yd, ad, dl, ul, hist, timing, M // 100, M // 100, ws=ws)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        hist.zero_()
        best, code = N.noscope_threshold_sweep(3, sd, zd, yd, ad, dl, ul, hist, timing, M // 100, M // 100,
                                               ws=ws)
    wall = (time.perf_counter() - t0) / reps
    # phase 1 alone: one event pair per call on the launching stream, median of 9
    st = torch.cuda.current_stream()
    per, host = [], []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record(st)
        N.noscope_threshold_sweep(1, sd, zd, yd, ad, dl, ul, hist, ws=ws, stream=st)
        e1.record(st)
        host.append(time.perf_counter() - h0)
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1))
    h_ms = statistics.median(per)
    out["sweep_1M"] = {"timing_ps_mse_snn_full": list(timing),
                       "wall_ms_incl_readback": round(wall * 1e3, 3), "hist_ms": round(h_ms, 4),
                       "hist_ms_max": round(max(per), 4), "host_ms_per_call": round(statistics.median(host) * 1e3, 4),
                       "records_per_s": round(M / wall, 1), "hist_GBps": round(M * 14 / h_ms / 1e6, 1),
                       "best": {k: best[k] for k in ("j", "l", "h", "feasible", "cost_ps", "uncertain")}}
    # Scale point: 1e9 records generated on device, histogram
    # phase timed.  Its bound is the shared memory, not HBM: per record two binary
    # searches over the candidate grids (scattered smem loads) and ~1.14 scattered
    # smem atomics.  Ceilings measured on B200 (tools/smem_atomic_bw.cu,
    # profiles/r02/smem_atomic_bw.txt): 5.28 random-address u32 atomics and 4.7
    # random loads per clock per SM; ncu counts 0.967 shared-memory wavefronts per
    # record for this kernel (profiles/r02/ncu_sweep_hist_v2.txt; 1.97 before the
    # searches moved to the Eytzinger layout), at most one per clock per SM ->
    # smem_wavefront_floor_ms.
    M9 = 1_000_000_000
    g = torch.Generator(device=device).manual_seed(4)
    y9 = (torch.rand(M9, device=device, generator=g) < 0.15).to(torch.uint8)
    s9 = torch.empty(M9, dtype=torch.float64, device=device).exponential_(0.05, generator=g)
    s9 += 40.0 * y9
    s9[torch.rand(M9, device=device, generator=g) < 0.05] = -float("inf")
    z9 = torch.randn(M9, device=device, generator=g).add_(-1.0).add_(2.5 * y9)
    a9 = torch.where(torch.isinf(s9), y9, torch.zeros_like(y9))
    n_h1 = int((a9 != y9).sum())
    dl9 = torch.from_numpy(sg.delta_grid(s9[:1_000_000].cpu().numpy(), 100)).to(device)
    for _ in range(2):
        N.noscope_threshold_sweep(1, s9, z9, y9, a9, dl9, ul, hist)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        N.noscope_threshold_sweep(1, s9, z9, y9, a9, dl9, ul, hist)
    e1.record()
    torch.cuda.synchronize()
    ms9 = e0.elapsed_time(e1) / 3
    clk = 1.965e9
    wf_floor = M9 * 0.967 / 148 / clk * 1e3
    at_floor = (M9 + n_h1) / 5.28 / 148 / clk * 1e3
    out["sweep_1e9_hist"] = {"records": M9, "ms": round(ms9, 3), "GBps": round(M9 * 14 / ms9 / 1e6, 1),
                             "frac_of_hbm": round(M9 * 14 / ms9 / 1e6 / measured_peaks()[0], 4),
                             "smem_atomics_per_record": round((M9 + n_h1) / M9, 3),
                             "smem_atomic_floor_ms": round(at_floor, 3),
                             "smem_wavefront_floor_ms": round(wf_floor, 3),
                             "frac_of_smem_wavefront_floor": round(wf_floor / ms9, 3),
                             "ceilings": "measured on B200: tools/smem_atomic_bw.cu + ncu wavefronts/record"}
    del s9, z9, y9, a9
    # compaction (H4) and routing (H6) scale points: at the webcam hour they are ~10 us
    # launches, so their HBM fraction is shown on 2^30 dispositions / 2^28 logits
    hbm = measured_peaks()[0]
    NC = 1 << 30
    dsp = torch.where(torch.rand(NC, device=device, generator=g) < 0.15,
                      torch.full((), 2, dtype=torch.uint8, device=device),
                      torch.full((), 1, dtype=torch.uint8, device=device))
    nf = int((dsp == 2).sum())
    cws = torch.empty(N.lib().noscope_compact_workspace_bytes(NC), dtype=torch.uint8, device=device)
    cout = (torch.empty(NC, dtype=torch.int32, device=device), torch.zeros(1, dtype=torch.int64, device=device))
    ms = _time_ms(lambda: N.noscope_compact_fired(dsp, ws=cws, out=cout))
    assert int(cout[1].item()) == nf
    byt = NC + 4 * nf                              # disposition read + index write
    out["compaction_2e30"] = {"frames": NC, "fired": nf, "ms": round(ms, 3), "GBps": round(byt / ms / 1e6, 1),
                              "frac_of_hbm": round(byt / ms / 1e6 / hbm, 4),
                              "algorithmic_bytes": byt}
    del dsp, cws, cout
    NR = 1 << 28
    zr = torch.randn(NR, device=device, generator=g)
    lo, hi = -0.5, 0.5
    nu = int(((zr >= lo) & (zr <= hi)).sum())
    rws = torch.empty(N.lib().noscope_route_workspace_bytes(NR), dtype=torch.uint8, device=device)
    rout = (torch.empty(NR, dtype=torch.uint8, device=device), torch.empty(NR, dtype=torch.int32, device=device),
            torch.zeros(1, dtype=torch.int64, device=device))
    ms = _time_ms(lambda: N.noscope_route_logits(lo, hi, zr, ws=rws, out=rout))
    assert int(rout[2].item()) == nu
    byt = 4 * NR + NR + 4 * nu                     # logits read + route write + uncertain index write
    out["routing_2e28"] = {"logits": NR, "uncertain": nu, "ms": round(ms, 3), "GBps": round(byt / ms / 1e6, 1),
                           "frac_of_hbm": round(byt / ms / 1e6 / hbm, 4), "algorithmic_bytes": byt}
    del zr, rws, rout
    return out


def _time_ms(fn, reps=3, rounds=5):
    """Median over `rounds` of the mean time of `reps` back-to-back calls (after one warm-up)."""
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(rounds):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return float(np.median(ts))


def tiny_config(device):
    """BASELINE configs[0]: 1,000 50x50 frames, global MSE vs the
    reference image, t_skip 1, L2C32D32, thresholds -2/+2 logits; launch-latency
    bound: median of 100 calls after 10 warm-ups, direct and CUDA-graph replay."""
    import torch
    import synthgen as sg
    from paper_1703_02529_b200 import noscope as N
    from synthgen.gpu import GpuScene, truth_labeller_address
    n = 1000
    sc = sg.make_scene(sg.SceneSpec(50, 50, n, seed=1, prevalence=0.15))
    gs = GpuScene(sc, device=device)
    fr = torch.empty((n, 7504), dtype=torch.uint8, device=device)
    gs.render(fr, 0, n)
    dd = N.DD(mode=0, metric=0, delta_diff=20.0, ref_image=torch.from_numpy(sg.background(sc.spec)).to(device))
    arch = sg.CnnArch(2, 32, 32)
    A, W = N.Arch(2, 32, 32), N.Weights(sg.he_normal_weights(arch, 1), device=device)
    st = N.noscope_stream_state_init(dd)
    ws = N.workspace(N.OP_CASCADE_RUN, dd, A, n, device=device)
    bufs = dict(labels=torch.zeros(n, dtype=torch.uint8, device=device))
    cur = torch.cuda.current_stream()

    def call(stream):
        N.noscope_cascade_run(dd, A, W, -2.0, 2.0, fr, 50, 50, st, truth_labeller_address(), gs.truth, ws=ws,
                              stream=stream, **bufs)

    def median_us(fn):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
        for _ in range(10):
            fn()
        for a, b in ev:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3

    side = torch.cuda.Stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        call(side)
    cur.wait_stream(side)
    us = median_us(lambda: call(cur))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call(torch.cuda.current_stream())
    us_g = median_us(g.replay)
    return {"frames": n, "us_direct_median": round(us, 1), "fps_direct": round(n / us * 1e6, 1),
            "us_graph_median": round(us_g, 1), "fps_graph": round(n / us_g * 1e6, 1)}


def next_rows_extras(device, sc, gs, small, n):
    """SURVEY 8(f) NEXT #1-#3 measured on the CNN-grid frames (50x50, 65,536):
    bytes are algorithmic (what the step must read)."""
    import torch
    import synthgen as sg
    from paper_1703_02529_b200 import noscope as N
    hbm, bf16 = measured_peaks()[:2]
    out = {}
    y = gs.truth[:n].contiguous()
    neg = int((y == 0).sum())
    ws = N.fit_workspace(1, 1, 7500, device)
    ref = torch.empty(7500, dtype=torch.uint8, device=device)
    ms = _time_ms(lambda: N.noscope_reference_image(small, y, ref_out=ref, ws=ws))
    gb = neg * 7500 / ms / 1e6
    out["reference_image"] = {"frames": n, "ms_incl_sync": round(ms, 4), "GBps": round(gb, 1),
                              "frac_of_hbm": round(gb / hbm, 4)}
    k, g = 30, 10
    dd = N.DD(mode=1, metric=1, grid=g, t_diff_frames=k, lr_weights=torch.ones(g * g, device=device))
    feats = torch.empty((n, g * g), dtype=torch.float64, device=device)
    ms = _time_ms(lambda: N.noscope_block_features(dd, small, feats=feats))
    gb = (n * 7500 * 2 + n * g * g * 8) / ms / 1e6
    out["block_features"] = {"frames": n, "ms": round(ms, 4), "GBps": round(gb, 1), "frac_of_hbm": round(gb / hbm, 4)}
    F = feats[k:].contiguous()
    t = (y[k:] != y[:-k]).to(torch.uint8).contiguous()
    wsl = N.fit_workspace(F.shape[0], g * g, 0, device)
    info = {}
    ms = _time_ms(lambda: N.noscope_lr_fit(F, t, ws=wsl, info=info), reps=2)
    # per Newton step: one gradient/Hessian pass (n * E^2 / 2 fp64 FMAs) + one trial pass
    E = g * g + 1
    fl = (info["iters"] + 1) * F.shape[0] * (E * E + 4 * E) * 2 / ms / 1e9
    out["lr_fit"] = {"examples": F.shape[0], "features": g * g, "newton_steps": info["iters"],
                     "grad_inf": info["grad_inf"], "stop": info["stop"], "ms_incl_sync": round(ms, 3),
                     "fp64_TFLOPs": round(fl, 2)}
    big = torch.randint(0, 2, (256 * 1024 * 1024,), dtype=torch.uint8, device=device)
    ref2 = big.roll(7)
    ms = _time_ms(lambda: N.noscope_eval_labels(big, ref2))
    gb = 2 * big.numel() / ms / 1e6
    out["eval_labels"] = {"frames": big.numel(), "ms_incl_sync": round(ms, 3), "GBps": round(gb, 1),
                          "frac_of_hbm": round(gb / hbm, 4)}
    del big, ref2
    # full CBO search: 2 DD configs x 2 CNNs on 16,384 evaluation frames
    m = 16384
    fr = small[:m]
    ym = y[:m]
    bg = torch.from_numpy(sg.background(sc.spec)).to(device)
    u = torch.linspace(-3, 3, 100, device=device, dtype=torch.float32)
    d0 = N.DD(mode=0, metric=0, ref_image=bg)
    d1 = N.DD(mode=1, metric=1, grid=10, t_diff_frames=30, lr_weights=torch.full((100,), 0.02, device=device),
              lr_bias=-1.0)
    dg = torch.logspace(-1, 4, 100, dtype=torch.float64, device=device)
    cnns = []
    for a in (sg.CnnArch(2, 32, 32), sg.CnnArch(4, 32, 32)):
        cnns.append((N.Arch(a.n_conv, a.base_filters, a.dense), N.Weights(sg.he_normal_weights(a, 3), device=device),
                     40 if a.n_conv == 2 else 100))
    ms = _time_ms(lambda: N.noscope_cbo_search([(d0, dg), (d1, dg)], cnns, fr, 50, 50, ym, u, 5, 12_500_000,
                                               m // 100, m // 100), reps=2)
    out["cbo_search"] = {"eval_frames": m, "dd_configs": 2, "cnns": 2, "ms_incl_sync": round(ms, 2)}
    # NEXT #4: specialized-CNN training, L2C32D32, 8,192 frames x 2 epochs, batch 64; the
    # GEMMs run on the tcgen05 tensor cores in 3xTF32 (three tf32 products per fp32
    # product): tensor rate = 3 x the algorithmic FLOP rate, against the tf32 dense peak
    # (the measured bf16 peak x the nominal tf32/bf16 ratio 0.5, B200_PROFILING.md)
    arch = sg.CnnArch(2, 32, 32)
    A = N.Arch(2, 32, 32)
    nt, ep = 8192, 2
    p = N.params_from_weight_dict(A, sg.he_normal_weights(arch, 3), device)
    perms = torch.stack([torch.randperm(nt, device=device) for _ in range(ep)]).to(torch.int32)
    val = torch.arange(nt, nt + 1024, dtype=torch.int32, device=device)
    N.noscope_cnn_train(A, p.clone(), small, y, perms[:1, :128].contiguous(), val[:64], batch=64)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hist, run = N.noscope_cnn_train(A, p, small, y, perms, val, batch=64)
    dt = time.perf_counter() - t0
    fwd = cnn_flops_per_frame((2, 32, 32))
    conv1 = 2 * 2500 * 27 * 32
    train_flops = (3 * fwd - conv1) * nt * run + fwd * 1024 * run     # fwd + dW + dX (no dX for conv1), + val
    tf32_peak = bf16 * 0.5   # TFLOP/s
    out["cnn_train"] = {"arch": "L2C32D32", "frames": nt, "epochs": run, "batch": 64, "s": round(dt, 3),
                        "frames_per_s": round(nt * run / dt, 1), "tflops": round(train_flops / dt / 1e12, 2),
                        "tensor_tflops_3xtf32": round(3 * train_flops / dt / 1e12, 2),
                        "frac_of_tf32_peak": round(3 * train_flops / dt / 1e12 / tf32_peak, 4),
                        "history": [[round(a, 5), round(b, 5)] for a, b in hist]}
    # live-stream latency: one 30-frame chunk (1 s of 30 fps video) per call, direct
    # vs replayed from a CUDA graph captured once (the chunk pipeline has no host sync)
    from synthgen.gpu import truth_labeller_address
    c = 30
    fr30 = small[:c].contiguous()
    y30 = y[:c].contiguous()
    arch = sg.CnnArch(2, 32, 32)
    A, Wt = N.Arch(2, 32, 32), N.Weights(sg.he_normal_weights(arch, 3), device=device)
    st = N.noscope_stream_state_init(d0)
    wsc = N.workspace(N.OP_CASCADE_RUN, d0, A, c, device=device)
    bufs = dict(labels=torch.zeros(c, dtype=torch.uint8, device=device),
                route_out=torch.zeros(c, dtype=torch.uint8, device=device))
    cur = torch.cuda.current_stream()
    call = lambda: N.noscope_cascade_run(d0, A, Wt, -0.05, 0.05, fr30, 50, 50, st, truth_labeller_address(), y30,
                                         ws=wsc, stream=cur, **bufs)
    side = torch.cuda.Stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        call()
    cur.wait_stream(side)
    ms_direct = _time_ms(call, reps=50)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        N.noscope_cascade_run(d0, A, Wt, -0.05, 0.05, fr30, 50, 50, st, truth_labeller_address(), y30, ws=wsc,
                              stream=torch.cuda.current_stream(), **bufs)
    ms_graph = _time_ms(graph.replay, reps=50)
    out["live_chunk_30"] = {"frames": c, "source": "50x50", "us_direct": round(ms_direct * 1e3, 1),
                            "us_graph_replay": round(ms_graph * 1e3, 1)}
    return out


def oracle_sample(S_or_none, frames_n):
    """Run the CPU oracle cascade on a bounded sample of the webcam workload."""
    import oracle as O
    import synthgen as sg
    t_begin = 50_000
    sc = sg.make_scene(sg.SceneSpec(W_SRC, H_SRC, UNIT, seed=2, stream=0))
    fr = sg.render_frames(sc, t_begin, t_begin + frames_n)
    src = fr[:, :W_SRC * H_SRC * 3].reshape(-1, H_SRC, W_SRC, 3)
    arch, w, (lr_w, lr_b) = make_weights()
    delta = S_or_none["dd"].delta_diff if S_or_none else -2.5
    lo = S_or_none["lo"] if S_or_none else -0.1
    hi = S_or_none["hi"] if S_or_none else 0.1
    cfg = O.DDConfig(mode=1, metric=1, out_w=OUT, out_h=OUT, grid=GRID, t_diff_frames=K_LAG,
                     t_skip_frames=1, delta_diff=delta, lr_w=lr_w, lr_b=lr_b)
    truth = sc.truth[t_begin:t_begin + frames_n]
    return src, cfg, arch, w, lo, hi, truth


def host_cpu():
    """nproc and the CPU model string of this host (lscpu, else /proc/cpuinfo)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")), None)
    except Exception:
        pass
    if model is None:
        try:
            model = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")),
                         None)
        except Exception:
            model = None
    return {"nproc": os.cpu_count(), "model": model}


def _pool(fn, jobs):
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        t0 = time.perf_counter()
        res = pool.map(fn, jobs)
        return res, time.perf_counter() - t0


def cpu_baseline(args, S):
    """The CPU oracle (oracle/, as it stands) on this host, SURVEY 8(d) "oracle timing":
    W (the metric's workload) on 1 core over a frame sample and on all cores over one
    13,500-frame unit; T, G and S legs on 1 core and on all cores.  Each leg states its
    sample; the main `value` is W on 1 core."""
    import oracle as O
    from threadpoolctl import threadpool_limits
    P = os.cpu_count() or 1
    delta, lo, hi = S["dd"].delta_diff, S["lo"], S["hi"]
    src, cfg, arch, w, _, _, truth = oracle_sample(S, args.cpu_frames)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        O.cascade(src, cfg, arch, w, lo, hi, truth)
        dt = time.perf_counter() - t0
    out = {"value": round(len(src) / dt, 3), "unit": "frames/s", "cores": 1, "kind": "oracle",
           "sample": f"{len(src)} consecutive frames (t=50000..) of the webcam unit processed as one "
                     f"unit by the plain CPU oracle (numpy, 1 thread), {dt:.1f} s; the oracle's per-frame "
                     f"work is position-independent, so the 13,500-frame W unit takes "
                     f"{13500 * dt / len(src):.0f} s on 1 core (extrapolated)",
           "host": host_cpu()}
    # W on all cores: the 13,500-frame unit (SURVEY 8(d) W "1 unit") as P contiguous segments,
    # each run as its own unit by one single-threaded process
    unit = 13_500
    b = np.linspace(0, unit, P + 1).astype(int)
    res, _ = _pool(_oracle_w_segment, [(delta, lo, hi, int(b[r]), int(b[r + 1])) for r in range(P)])
    slow = max(res)
    out["all_cores"] = {"value": round(unit / slow, 3), "cores": P,
                        "sample": f"one 13,500-frame W unit (frames 0..13499 of stream 0) split into {P} "
                                  f"contiguous segments, one single-threaded process each (each segment "
                                  f"starts a unit: its first 30 checked frames are forced fires); time = "
                                  f"the slowest process's oracle time, {slow:.1f} s (process start and "
                                  f"input rendering excluded)"}
    out["legs"] = oracle_legs(P)
    return out


def _oracle_w_segment(a):
    delta, lo, hi, t0, t1 = a
    import oracle as O
    import synthgen as sg
    from threadpoolctl import threadpool_limits
    sc = sg.make_scene(sg.SceneSpec(W_SRC, H_SRC, UNIT, seed=2, stream=0))
    fr = sg.render_frames(sc, t0, t1)
    src = fr[:, :W_SRC * H_SRC * 3].reshape(-1, H_SRC, W_SRC, 3)
    arch, w, (lr_w, lr_b) = make_weights()
    cfg = O.DDConfig(mode=1, metric=1, out_w=OUT, out_h=OUT, grid=GRID, t_diff_frames=K_LAG,
                     t_skip_frames=1, delta_diff=delta, lr_w=lr_w, lr_b=lr_b)
    with threadpool_limits(1):
        st = time.perf_counter()
        O.cascade(src, cfg, arch, w, lo, hi, sc.truth[t0:t1])
        return time.perf_counter() - st


def _tiny_inputs(t0=0, t1=1000):
    import synthgen as sg
    sc = sg.make_scene(sg.SceneSpec(50, 50, 1000, seed=1))
    fr = sg.render_frames(sc, t0, t1)[:, :7500].reshape(-1, 50, 50, 3)
    return sc, fr


def _oracle_t_job(a):
    """T: tiny cascade (global MSE vs the reference image, delta 20, L2C32D32, -2/+2)."""
    t0, t1 = a
    import oracle as O
    import synthgen as sg
    from threadpoolctl import threadpool_limits
    sc, fr = _tiny_inputs(t0, t1)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 1)
    cfg = O.DDConfig(mode=0, metric=0, delta_diff=20.0, ref_image=sg.background(sc.spec))
    with threadpool_limits(1):
        st = time.perf_counter()
        O.cascade(fr, cfg, arch, w, -2.0, 2.0, sc.truth[t0:t1])
        return time.perf_counter() - st


def _oracle_g_job(a):
    """G: the CNN on frames [f0, f1) of the 65,536-frame grid input, one architecture."""
    ai, f0, f1 = a
    import oracle as O
    import synthgen as sg
    from threadpoolctl import threadpool_limits
    arch = sg.ARCH_GRID[ai]
    sc = sg.make_scene(sg.SceneSpec(50, 50, 65536, seed=3, prevalence=0.15))
    g = sg.render_frames(sc, f0, f1)[:, :7500].reshape(-1, 50, 50, 3)
    w = sg.he_normal_weights(arch, 3)
    with threadpool_limits(1):
        st = time.perf_counter()
        O.cnn_logits(g, arch, w)
        return time.perf_counter() - st


def _sweep_records_1m():
    """The bench's 1M-record sweep instance (config S) and its 100 x 100 candidates."""
    import synthgen as sg
    rng = np.random.default_rng(4)
    M = 1_000_000
    y = (rng.random(M) < 0.15).astype(np.uint8)
    s = np.where(rng.random(M) < 0.05, -np.inf, rng.gamma(2.0, 10.0, M) + 40.0 * y)
    z = (rng.normal(0, 1, M) + 2.5 * y - 1.0).astype(np.float32)
    a_ = np.where(np.isinf(s), y, 0).astype(np.uint8)
    return s, z, y, a_, sg.delta_grid(s, 100), sg.logit_grid(100)


def _oracle_s_job(a):
    """S: the oracle's direct per-threshold tables over records [r0, r1)."""
    r0, r1 = a
    import oracle as O
    from threadpoolctl import threadpool_limits
    s, z, y, a_, dl, ul = _sweep_records_1m()
    with threadpool_limits(1):
        st = time.perf_counter()
        T = O.sweep_tables(s[r0:r1], z[r0:r1], y[r0:r1], a_[r0:r1], dl, ul)
        return time.perf_counter() - st, T


def oracle_legs(P):
    """T / G / S oracle timings, 1 core and all cores."""
    import oracle as O
    import synthgen as sg
    legs = {}
    # T: all 1,000 frames
    t1 = _oracle_t_job((0, 1000))
    b = np.linspace(0, 1000, P + 1).astype(int)
    res, _ = _pool(_oracle_t_job, [(int(b[r]), int(b[r + 1])) for r in range(P)])
    legs["T"] = {"frames": 1000, "one_core_fps": round(1000 / t1, 1), "all_cores_fps": round(1000 / max(res), 1),
                 "sample": "all 1,000 tiny frames; all cores = mode-0 frames split into P independent "
                           "segments (exact: mode 0 has no cross-frame state); time = slowest process's "
                           "oracle time (process start and rendering excluded)"}
    # G: 1,024 frames per architecture on all cores; 64 per architecture on 1 core
    flops = sum(cnn_flops_per_frame((a.n_conv, a.base_filters, a.dense)) for a in sg.ARCH_GRID)
    one = [_oracle_g_job((ai, 0, 64)) for ai in range(len(sg.ARCH_GRID))]
    per = max(1, P // len(sg.ARCH_GRID))
    fb = np.linspace(0, 1024, per + 1).astype(int)
    res, _ = _pool(_oracle_g_job, [(ai, int(fb[k]), int(fb[k + 1])) for ai in range(len(sg.ARCH_GRID))
                                   for k in range(per)])
    wall = max(res)
    legs["G"] = {"one_core": {"frames_per_arch": 64,
                              "fps_per_arch": {a.name: round(64 / t, 1) for a, t in zip(sg.ARCH_GRID, one)},
                              "GFLOPs": round(64 * flops / sum(one) / 1e9, 2)},
                 "all_cores": {"frames_per_arch": 1024, "wall_s": round(wall, 2),
                               "fps_all_archs": round(1024 * len(sg.ARCH_GRID) / wall, 1),
                               "GFLOPs": round(1024 * flops / wall / 1e9, 2)},
                 "sample": "8 archs x 1,024 frames on all cores (frames split per arch into "
                           f"{per} slices, one single-threaded process each; time = slowest process); "
                           "64 frames per arch on 1 core"}
    # S: 1M records, 100 x 100 candidates; 1 core on a 100k-record prefix (the direct
    # tables are linear in the records) + the full triple search; all cores on all 1M
    (t_tab, T1), = [_oracle_s_job((0, 100_000))]
    st = time.perf_counter()
    O.sweep_best(T1, SWEEP_TIMING, 1000, 1000)
    t_best = time.perf_counter() - st
    rb = np.linspace(0, 1_000_000, P + 1).astype(int)
    res, _ = _pool(_oracle_s_job, [(int(rb[r]), int(rb[r + 1])) for r in range(P)])
    st = time.perf_counter()
    T = {k: sum(r[1][k] for r in res) for k in res[0][1]}
    O.sweep_best(T, SWEEP_TIMING, 10_000, 10_000)
    wall = max(r[0] for r in res) + time.perf_counter() - st
    legs["S"] = {"records": 1_000_000, "candidates": [100, 100],
                 "one_core_s_extrapolated": round(t_tab * 10 + t_best, 2),
                 "one_core_records_per_s": round(1_000_000 / (t_tab * 10 + t_best), 1),
                 "all_cores_s": round(wall, 2), "all_cores_records_per_s": round(1_000_000 / wall, 1),
                 "sample": "1 core: direct per-(j, t) tables over a 100,000-record prefix (x10, tables are "
                           "linear in the records) + the full 505,000-triple search; all cores: tables of "
                           "P record shards summed (integer counts) + the search"}
    return legs


def run_reference(args):
    """Reference arm: the oracle as it stands, on a bounded sample per step."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    from threadpoolctl import threadpool_limits
    per_step = 96
    src, cfg, arch, w, lo, hi, truth = oracle_sample(None, per_step)
    with threadpool_limits(1):
        for _ in range(args.warmup):
            O.cascade(src, cfg, arch, w, lo, hi, truth)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            O.cascade(src, cfg, arch, w, lo, hi, truth)
        dt = (time.perf_counter() - t0) / args.steps
    v = round(per_step / dt, 3)
    line = {"impl": "reference", "metric": "cascade frames/sec (diff+CNN+routing)", "value": v,
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64/f64 (numpy oracle)", "data": "synthetic",
            "config": {"workload": CONFIG_NAME, "sample_frames_per_step": per_step},
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": 1, "kind": "oracle",
                             "sample": f"{per_step} frames of the webcam unit per step"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        maybe_self_launch(a)
        if a.workload == "x":
            run_x(a)
        else:
            run_ours(a)
