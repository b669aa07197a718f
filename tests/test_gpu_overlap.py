"""The overlapped cascade schedule (noscope_api.cu cascade_front_overlapped, opt-in
with NOSCOPE_OVERLAP=1): for calls of >= 8,192 frames on the band-pipeline DD with a
conv2-fused L = 2 CNN, the conv1+conv2 kernel runs on a few SMs beside dd_kernel,
consuming a queue of fired frames while the DD streams, and a whole-GPU launch
finishes the rest.

Its results must be those of the serial schedule (NOSCOPE_OVERLAP=0), bit for bit —
labels, routes, logits, scores and run counts — whatever the side-SM budget
(which moves the split between the side and the tail launch) and the chunking; and
the oracle (O1-O8) recomputes sampled frames one by one, so the overlap path is
pinned to the paper's arithmetic directly as well as through the serial schedule
(itself parity-tested in test_gpu_cascade.py / test_gpu_fullsize.py)."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import ns, requires_gpu

pytestmark = [pytest.mark.gpu, requires_gpu]

W, H = 640, 480


class _env:
    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _video(n, seed, prevalence):
    from synthgen.gpu import GpuScene
    sc = sg.make_scene(sg.SceneSpec(W, H, n, seed=seed, prevalence=prevalence))
    gs = GpuScene(sc)
    frames = torch.empty((n, sg.frame_pitch(W, H)), dtype=torch.uint8, device="cuda")
    for t0 in range(0, n, 4096):
        gs.render(frames[t0:t0 + 4096], t0, min(4096, n - t0))
    return sc, gs, frames


def _run(nsm, dd, arch, w, lo, hi, frames, gs, chunks):
    from synthgen.gpu import truth_labeller_address
    n = frames.shape[0]
    state = nsm.noscope_stream_state_init(dd)
    out = {"labels": [], "route": [], "logits": [], "scores": [], "stats": []}
    pos = 0
    for c in chunks:
        r = torch.zeros(c, dtype=torch.uint8, device="cuda")
        z = torch.full((c,), float("nan"), device="cuda")
        s = torch.zeros(c, dtype=torch.float64, device="cuda")
        o = nsm.noscope_cascade_run(dd, nsm.Arch(arch.n_conv, arch.base_filters, arch.dense), nsm.Weights(w),
                                    lo, hi, frames[pos:pos + c], W, H, state, truth_labeller_address(),
                                    gs.truth, seg_offset=pos, frame_index_base=pos, route_out=r,
                                    logits_out=z, scores_out=s, want_stats=True)
        torch.cuda.synchronize()
        out["labels"].append(o["labels"][:c].cpu().numpy())
        out["route"].append(r.cpu().numpy())
        out["logits"].append(z.cpu().numpy())
        out["scores"].append(s.cpu().numpy())
        out["stats"].append(dict(o["stats"]))
        pos += c
    assert pos == n
    for k in ("labels", "route", "logits", "scores"):
        out[k] = np.concatenate(out[k])
    return out


def _same(a, b):
    assert np.array_equal(a["scores"], b["scores"])
    assert np.array_equal(a["route"], b["route"])
    assert np.array_equal(a["labels"], b["labels"])
    # logits are written for fired frames only (NaN elsewhere in both)
    assert np.array_equal(a["logits"].view(np.uint32), b["logits"].view(np.uint32))
    assert a["stats"] == b["stats"]


def _oracle_samples(sc, out, dd_o, arch, w, k, samples):
    """Recompute sampled frames with the oracle: score bit-exact, disposition, and
    (for fired frames) the CNN logit within 2e-2."""
    bg = sg.background(sc.spec)
    fired = []
    for t in samples:
        G = O.downsample(sg.render_frame(sc, t, bg)[None], 50, 50)[0]
        if dd_o.mode == 1:
            if t < k:
                continue
            A = O.downsample(sg.render_frame(sc, t - k, bg)[None], 50, 50)[0]
        else:
            A = dd_o.ref_image
        s = O.score_frame(G, A, dd_o.metric, dd_o.grid, dd_o.lr_w, dd_o.lr_b)
        assert out["scores"][t] == s, t
        assert (out["route"][t] >= O.R_NEG) == (s > dd_o.delta_diff), t
        if out["route"][t] >= O.R_NEG:
            fired.append((t, G))
    assert fired
    z_o = O.cnn_logits(np.stack([g for _, g in fired]), arch, w)
    z_g = np.array([out["logits"][t] for t, _ in fired])
    assert np.abs(z_g - z_o).max() <= 2e-2


@pytest.mark.parametrize("base_filters,side,chunks,t_skip", [
    (32, 8, [24000], 1),            # the bench's schedule
    (32, 1, [24000], 1),            # slow side: most frames left to the tail launch
    (32, 32, [13000, 11000], 1),    # wide side; two chunks with carried state (both >= 8,192)
    (16, 8, [24000], 1),            # the paper's C = 16 models
    (32, 8, [14000, 13001], 3),     # frame skipping: t-30 anchors on checked frames, deferred fires
])
def test_overlap_equals_serial_blocked_lag(base_filters, side, chunks, t_skip):
    nsm = ns()
    n, k = sum(chunks), 30
    sc, gs, frames = _video(n, seed=5, prevalence=0.5)
    lr_w, lr_b = sg.lr_weights(10, 3)
    arch = sg.CnnArch(2, base_filters, 32)
    w = sg.he_normal_weights(arch, 4)
    delta = 2160.0
    dd = nsm.DD(mode=1, metric=1, grid=10, t_diff_frames=k, t_skip_frames=t_skip, delta_diff=delta,
                lr_weights=torch.from_numpy(lr_w).cuda(), lr_bias=float(lr_b))
    lo, hi = 0.0107, 0.1035
    with _env(NOSCOPE_OVERLAP=0):
        ser = _run(nsm, dd, arch, w, lo, hi, frames, gs, chunks)
    with _env(NOSCOPE_OVERLAP=1, NOSCOPE_SIDE_SMS=side):
        ovl = _run(nsm, dd, arch, w, lo, hi, frames, gs, chunks)
    nf = sum(s["n_fired"] for s in ovl["stats"])
    assert 0.05 * n / t_skip < nf < 0.95 * n / t_skip, nf   # a real queue, not a degenerate one
    _same(ovl, ser)
    del frames
    torch.cuda.empty_cache()
    dd_o = O.DDConfig(mode=1, metric=1, grid=10, t_diff_frames=k, t_skip_frames=t_skip, delta_diff=delta,
                      lr_w=lr_w, lr_b=lr_b)
    rng = np.random.default_rng(1)
    samples = sorted(set([k, k + 1, n - 1, chunks[0] - 1, min(chunks[0], n - 1)] +
                         rng.integers(k, n, 14 * t_skip).tolist()))
    samples = [t for t in samples if t % t_skip == 0]   # checked frames (skipped ones have no score)
    _oracle_samples(sc, ovl, dd_o, arch, w, k, samples)


@pytest.mark.parametrize("delta", [-np.inf, np.inf])
def test_overlap_all_or_nothing_fired(delta):
    """Every checked frame fired (the queue holds the whole call) and none fired
    (an empty queue: only the tail launch's claims, all failing)."""
    nsm = ns()
    n = 9000
    sc, gs, frames = _video(n, seed=6, prevalence=0.3)
    ref = sg.background(sc.spec)
    ref_s = O.downsample(ref[None], 50, 50)[0]
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 2)
    dd = nsm.DD(mode=0, metric=0, t_skip_frames=2, delta_diff=float(delta),
                ref_image=torch.from_numpy(np.ascontiguousarray(ref_s)).cuda())
    with _env(NOSCOPE_OVERLAP=0):
        ser = _run(nsm, dd, arch, w, -1.0, 1.0, frames, gs, [n])
    with _env(NOSCOPE_OVERLAP=1):
        ovl = _run(nsm, dd, arch, w, -1.0, 1.0, frames, gs, [n])
    _same(ovl, ser)
    want = (n + 1) // 2 if delta < 0 else 0         # t_skip 2: frames 0, 2, 4, ...
    assert ovl["stats"][0]["n_fired"] == want
    if delta < 0:   # the oracle's logits of a sample of the fired frames
        bg = sg.background(sc.spec)
        ts = [0, 2, 4000, n - 1 - ((n - 1) % 2)]
        G = np.stack([O.downsample(sg.render_frame(sc, t, bg)[None], 50, 50)[0] for t in ts])
        z_o = O.cnn_logits(G, arch, w)
        assert np.abs(ovl["logits"][ts] - z_o).max() <= 2e-2
