"""Multi-GPU driver: one process per GPU (torchrun), units sharded by rank.

Units (stream x time segment) are independent, so the cascade
itself has no collective; the two exchanges the north star names are
  C1  all_reduce(SUM) of the sweep histogram between phase 1 and phase 2
      (integer counts -> bit-identical for every world size), and
  C2  gather of the per-unit label tracks to rank 0.
Works with NCCL (GPU tensors) and gloo (CPU tensors, used by the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def unit_range(n_units: int, world: int, rank: int):
    """Contiguous block of units for `rank`: [r*U/G, (r+1)*U/G)."""
    return (rank * n_units) // world, ((rank + 1) * n_units) // world


def world_rank():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def allreduce_hist_(hist: torch.Tensor) -> torch.Tensor:
    """C1: in-place sum of a uint64-count histogram (stored as int64) over ranks
    (a collective whenever a process group exists, also with one rank)."""
    if dist.is_available() and dist.is_initialized():
        if hist.device.type == "cuda" and dist.get_backend() != "nccl":   # gloo: reduce a host copy
            h = hist.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM)
            hist.copy_(h)
        else:
            dist.all_reduce(hist, op=dist.ReduceOp.SUM)
    return hist


def gather_labels(local: torch.Tensor, counts=None):
    """C2 (all ranks receive): concatenate every rank's label track in rank order.

    `counts` (list of per-rank lengths) allows unequal shards; default equal."""
    world, _ = world_rank()
    if world == 1:
        return local
    if counts is None:
        counts = [local.numel()] * world
    m = max(counts)
    buf = torch.zeros(m, dtype=local.dtype, device=local.device)
    buf[:local.numel()] = local
    if local.device.type == "cuda" and dist.get_backend() == "nccl":
        out = torch.empty(m * world, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, buf)
        parts = list(out.view(world, m))
    else:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def gather_labels_to_rank0(local: torch.Tensor, out: torch.Tensor | None = None):
    """C2: per-unit label tracks gathered to rank 0 only (dist.gather; NCCL or gloo).
    Every rank passes an equal-length track; rank 0 returns the concatenation in
    rank order (written into `out` [world * n] if given), other ranks None."""
    world, rank = world_rank()
    if not (dist.is_available() and dist.is_initialized()):
        if out is not None:
            out.copy_(local)
            return out
        return local
    staged = local.device.type == "cuda" and dist.get_backend() != "nccl"   # gloo gathers host tensors
    src = local.cpu() if staged else local
    if rank == 0:
        out = out if out is not None else torch.empty(world * local.numel(), dtype=local.dtype,
                                                      device=local.device)
        tgt = torch.empty(world * local.numel(), dtype=local.dtype) if staged else out
        dist.gather(src, gather_list=list(tgt.view(world, local.numel())), dst=0)
        if staged:
            out.copy_(tgt)
        return out
    dist.gather(src, dst=0)
    return None


def distributed_sweep(hist_fn, evaluate_fn, n_words: int, device):
    """Phase 1 on the local shard (hist_fn(hist) accumulates into a zeroed
    histogram), C1 all-reduce, then phase 2 (evaluate_fn(hist)) — identical on
    every rank because the summed counts are identical."""
    hist = torch.zeros(n_words, dtype=torch.int64, device=device)
    hist_fn(hist)
    allreduce_hist_(hist)
    return evaluate_fn(hist), hist


def sweep_on_shard(nsm, s, z, y, a, delta, u, timing, fp_limit, fn_limit):
    """The GPU path: noscope_threshold_sweep phase 1 locally, allreduce, phase 2."""
    n_words = nsm.sweep_hist_words(delta.numel(), u.numel())

    def hist_fn(h):
        nsm.noscope_threshold_sweep(1, s, z, y, a, delta, u, h)

    def eval_fn(h):
        return nsm.noscope_threshold_sweep(2, None, None, None, None, delta, u, h, timing, fp_limit,
                                           fn_limit)

    (best, code), _ = distributed_sweep(hist_fn, eval_fn, n_words, delta.device)
    return best, code


def run_units(nsm, units, make_frames, dd, arch, weights, lo, hi, labeller, labeller_user_fn,
              chunk=8192, ws=None, device="cuda", timer=None, records=None):
    """Process this rank's units through noscope_cascade_run in chunks with
    carried stream state (R-19: no state crosses a unit boundary); returns the
    concatenated label track.

    make_frames(u, t0, m) -> device frames of unit u, ordinals [t0, t0+m) (the
    decode stand-in; called outside the timed intervals).  timer: optional list;
    a (start, end) CUDA event pair is appended around every cascade call, so the
    caller can sum the cascade time without the generation.  records: optional
    dict of per-unit lists that receives each unit's scores / logits (device); if it
    holds "flat" = (scores, logits) tensors of all units' frames, the per-unit records
    are consecutive slices of those (one sweep call can then cover every unit)."""
    outs = []
    off = 0
    for u in units:
        n = u["n_frames"]
        state = nsm.noscope_stream_state_init(dd)
        labels = torch.empty(n, dtype=torch.uint8, device=device)
        scores = logits = None
        if records is not None and "flat" in records:
            scores, logits = records["flat"][0][off:off + n], records["flat"][1][off:off + n]
        elif records is not None:
            scores = torch.empty(n, dtype=torch.float64, device=device)
            logits = torch.zeros(n, dtype=torch.float32, device=device)
        off += n
        for t0 in range(0, n, chunk):
            m = min(chunk, n - t0)
            frames = make_frames(u, t0, m)
            if timer is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            nsm.noscope_cascade_run(dd, arch, weights, lo, hi, frames, u["width"], u["height"], state,
                                    labeller, labeller_user_fn(u), seg_offset=t0,
                                    frame_index_base=t0, ws=ws, labels=labels[t0:t0 + m],
                                    scores_out=None if scores is None else scores[t0:t0 + m],
                                    logits_out=None if logits is None else logits[t0:t0 + m])
            if timer is not None:
                ev[1].record()
                timer.append(ev)
        if records is not None:
            records.setdefault("scores", []).append(scores)
            records.setdefault("logits", []).append(logits)
        outs.append(labels)
    return torch.cat(outs) if outs else torch.empty(0, dtype=torch.uint8, device=device)
