"""GPU parity: downsample + difference detector + compaction (noscope_diff_detect)
against the oracle on the same seeded inputs.  Dispositions and compaction are
compared bit-exact, downsampled frames byte-exact, scores to rel 1e-5 (the
north-star bound; the implementation is expected to be exactly equal)."""
import functools
import math

import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import dd_pair, hw3, ns, requires_gpu, scene_frames

pytestmark = [pytest.mark.gpu, requires_gpu]


def _run(nsm, g, frames_np, W, H, seg_offset=0, state=None):
    fr = torch.from_numpy(frames_np).cuda()
    out = nsm.noscope_diff_detect(g, fr, W, H, seg_offset=seg_offset, state=state)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in out.items()}


def _compare(res, small_o, score_o, disp_o, out=50, needed=None):
    n = len(disp_o)
    assert np.array_equal(res["disp"][:n], disp_o)
    idx_o = O.compact(disp_o)
    assert int(res["n_fired"][0]) == len(idx_o)
    assert np.array_equal(res["idx"][:len(idx_o)], idx_o)
    s_g, s_o = res["score"][:n], score_o
    fin = np.isfinite(s_o)
    assert np.array_equal(np.isinf(s_g), np.isinf(s_o)) and np.array_equal(s_g[~fin], s_o[~fin])
    assert np.allclose(s_g[fin], s_o[fin], rtol=1e-5, atol=1e-12)
    assert np.array_equal(s_g[fin], s_o[fin]), "expected exact fp64 scores"
    sb = out * out * 3
    rows = np.arange(n) if needed is None else needed
    assert np.array_equal(res["small"][rows, :sb], small_o.reshape(n, -1)[rows])


def test_synthgen_gpu_matches_cpu():
    from synthgen.gpu import GpuScene
    for (W, H, n) in [(50, 50, 40), (640, 480, 6), (101, 77, 9)]:
        sc, fr = scene_frames(W, H, n, seed=5, prevalence=0.9)
        gs = GpuScene(sc)
        out = torch.zeros((n, fr.shape[1]), dtype=torch.uint8, device="cuda")
        gs.render(out, 0, n)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), fr)


@pytest.mark.parametrize("n", [1, 37, 1000, 4097])
def test_tiny_global_vs_reference_image(n):
    nsm = ns()
    sc, fr = scene_frames(50, 50, n, seed=1, prevalence=0.3)
    ref = sg.background(sc.spec)
    ocfg, g = dd_pair(nsm, 0, 0, delta=20.0, ref=ref)
    small = hw3(fr, 50, 50)
    s_o, d_o = O.diff_detect(small, ocfg)
    res = _run(nsm, g, fr, 50, 50)
    _compare(res, small, s_o, d_o)


@pytest.mark.parametrize("mode,metric,t_skip", [(0, 1, 1), (1, 0, 1), (1, 1, 1), (1, 1, 4), (0, 0, 3)])
def test_webcam_640x480(mode, metric, t_skip):
    nsm = ns()
    n = 70
    sc, fr = scene_frames(640, 480, n, seed=2, prevalence=0.95)
    src = hw3(fr, 640, 480)
    small_o = O.downsample(src, 50, 50)
    lr = sg.lr_weights(10, 3)
    ref = O.downsample(sg.background(sc.spec)[None], 50, 50)[0]
    s_tmp, _ = O.diff_detect(small_o, O.DDConfig(mode=mode, metric=metric, grid=10, t_diff_frames=7,
                                                 t_skip_frames=t_skip, delta_diff=0.0,
                                                 ref_image=ref, lr_w=lr[0], lr_b=lr[1]))
    fin = s_tmp[np.isfinite(s_tmp)]
    delta = float(np.quantile(fin, 0.5)) if fin.size else 0.0
    ocfg, g = dd_pair(nsm, mode, metric, k=7, t_skip=t_skip, delta=delta, ref=ref, lr=lr)
    s_o, d_o = O.diff_detect(small_o, ocfg)
    assert 0 < (d_o == O.FIRED).sum() < n
    res = _run(nsm, g, fr, 640, 480)
    # small frames are written for checked frames and (mode 1) anchors only
    need = [t for t in range(n) if t % t_skip == 0 or (mode == 1 and (t + 7) % t_skip == 0)]
    _compare(res, small_o, s_o, d_o, needed=np.array(need))


@pytest.mark.parametrize("t_skip,chunks", [(1, [23, 1, 40, 6]), (3, [10, 11, 49]), (4, [7, 63])])
def test_chunked_with_state_equals_whole_unit(t_skip, chunks):
    nsm = ns()
    n = sum(chunks)
    sc, fr = scene_frames(160, 120, n, seed=4, prevalence=0.9)
    small_o = O.downsample(hw3(fr, 160, 120), 50, 50)
    lr = sg.lr_weights(10, 5)
    ocfg, g = dd_pair(nsm, 1, 1, k=9, t_skip=t_skip, delta=-3.9, lr=lr)
    s_o, d_o = O.diff_detect(small_o, ocfg)
    state = nsm.noscope_stream_state_init(g)
    pos = 0
    disp = np.empty(n, np.uint8)
    score = np.empty(n)
    for c in chunks:
        r = _run(nsm, g, fr[pos:pos + c], 160, 120, seg_offset=pos, state=state)
        disp[pos:pos + c] = r["disp"][:c]
        score[pos:pos + c] = r["score"][:c]
        pos += c
    assert np.array_equal(disp, d_o)
    assert np.array_equal(score, s_o)


def test_odd_width_generic_path_and_identity():
    nsm = ns()
    for (W, H, out) in [(101, 77, 50), (50, 50, 50), (53, 61, 17)]:
        sc, fr = scene_frames(W, H, 30, seed=6, prevalence=0.8)
        small_o = O.downsample(hw3(fr, W, H), out, out)
        ocfg, g = dd_pair(nsm, 1, 0, out=out, k=2, delta=3.0)
        s_o, d_o = O.diff_detect(small_o, ocfg)
        res = _run(nsm, g, fr, W, H)
        _compare(res, small_o, s_o, d_o, out=out)


def test_extreme_deltas_and_identical_frames():
    nsm = ns()
    sc, fr = scene_frames(50, 50, 64, seed=7, prevalence=0.0, sigma=0)
    ref = sg.background(sc.spec)
    for delta, expect in [(math.inf, O.SUPPRESSED), (0.0, O.SUPPRESSED), (-math.inf, O.FIRED)]:
        ocfg, g = dd_pair(nsm, 0, 0, delta=delta, ref=ref)
        res = _run(nsm, g, fr, 50, 50)
        assert np.all(res["disp"][:64] == expect)


def test_validation_errors():
    nsm = ns()
    fr = torch.zeros((4, 7504), dtype=torch.uint8, device="cuda")
    _, g = dd_pair(nsm, 1, 0, out=60)
    with pytest.raises(nsm.NoScopeError) as e:
        nsm.noscope_diff_detect(g, fr, 50, 50)           # out > source
    assert e.value.code == 2
    _, g = dd_pair(nsm, 1, 0)
    with pytest.raises(nsm.NoScopeError):
        nsm.noscope_diff_detect(g, fr[:, :7500], 50, 50)  # pitch not /16


@functools.lru_cache(maxsize=None)
def _geom_frames(W, H, out):
    # 640x480: ~1.4 frames per CTA, so t-5 anchors sit several CTAs back (deferred path)
    n = {640: 200, 101: 3000, 160: 1200}[W]
    sc, fr = scene_frames(W, H, n, seed=11, prevalence=0.6)
    return fr, O.downsample(hw3(fr, W, H), out, out)


@pytest.mark.parametrize("ng,cps", [(1, 1), (2, 1), (3, 1), (5, 1), (2, 2)])
@pytest.mark.parametrize("geom", [(640, 480, 50, 1, 1), (101, 77, 23, 1, 0), (160, 120, 50, 0, 1)])
def test_dd_kernel_launch_geometries(monkeypatch, ng, cps, geom):
    """dd_kernel parity for every worker-group count / CTAs-per-SM the launch can take
    (the default is NG = 4, 1 CTA/SM): band ring per group, segment warps, scorer and
    deferred-anchor scoring must give the same bytes and scores in every geometry."""
    W, H, out, mode, metric = geom
    monkeypatch.setenv("NOSCOPE_DD_NG", str(ng))
    monkeypatch.setenv("NOSCOPE_DD_CPS", str(cps))
    nsm = ns()
    fr, small_o = _geom_frames(W, H, out)
    n = fr.shape[0]
    grid = 10 if out % 10 == 0 else 4
    lr = sg.lr_weights(grid, 7)
    ref = small_o[0].copy()
    cfg0 = O.DDConfig(mode=mode, metric=metric, out_w=out, out_h=out, grid=grid, t_diff_frames=5,
                      t_skip_frames=1, delta_diff=0.0, ref_image=ref, lr_w=lr[0], lr_b=lr[1])
    s_tmp, _ = O.diff_detect(small_o, cfg0)
    fin = s_tmp[np.isfinite(s_tmp)]
    delta = float(np.quantile(fin, 0.5))
    ocfg, g = dd_pair(nsm, mode, metric, out=out, grid=grid, k=5, t_skip=1, delta=delta, ref=ref, lr=lr)
    s_o, d_o = O.diff_detect(small_o, ocfg)
    res = _run(nsm, g, fr, W, H)
    _compare(res, small_o, s_o, d_o, out=out)


@pytest.mark.parametrize("mode,metric,t_skip,k", [(0, 0, 1, 1), (0, 1, 3, 1), (1, 0, 1, 1), (1, 1, 1, 30),
                                                  (1, 1, 4, 7), (1, 0, 3, 2)])
@pytest.mark.parametrize("size,grid", [(50, 10), (23, 4)])
def test_identity_downsample_path(mode, metric, t_skip, k, size, grid):
    """out == source size (BASELINE configs[0]): the identity kernel (source frame = small
    frame, t-k anchors read straight from the source frames), whole unit and in chunks
    with carried state (anchors from the state ring)."""
    nsm = ns()
    n = 1500
    sc, fr = scene_frames(size, size, n, seed=13, prevalence=0.4)
    small_o = hw3(fr, size, size)
    lr = sg.lr_weights(grid, 9)
    ref = sg.background(sc.spec)
    cfg0 = O.DDConfig(mode=mode, metric=metric, out_w=size, out_h=size, grid=grid, t_diff_frames=k,
                      t_skip_frames=t_skip, delta_diff=0.0, ref_image=ref, lr_w=lr[0], lr_b=lr[1])
    s_tmp, _ = O.diff_detect(small_o, cfg0)
    fin = s_tmp[np.isfinite(s_tmp)]
    delta = float(np.quantile(fin, 0.5))
    ocfg, g = dd_pair(nsm, mode, metric, out=size, grid=grid, k=k, t_skip=t_skip, delta=delta, ref=ref, lr=lr)
    s_o, d_o = O.diff_detect(small_o, ocfg)
    assert 0 < (d_o == O.FIRED).sum() < n
    need = [t for t in range(n) if t % t_skip == 0 or (mode == 1 and (t + k) % t_skip == 0)]
    res = _run(nsm, g, fr, size, size)
    _compare(res, small_o, s_o, d_o, out=size, needed=np.array(need))
    state = nsm.noscope_stream_state_init(g)
    disp = np.empty(n, np.uint8)
    score = np.empty(n)
    pos = 0
    for c in (1, 499, 3, 997):
        r = _run(nsm, g, fr[pos:pos + c], size, size, seg_offset=pos, state=state)
        disp[pos:pos + c] = r["disp"][:c]
        score[pos:pos + c] = r["score"][:c]
        pos += c
    assert np.array_equal(disp, d_o)
    assert np.array_equal(score[np.isfinite(s_o)], s_o[np.isfinite(s_o)])


@pytest.mark.parametrize("W,H", [(1280, 720), (1170, 1080), (1000, 570), (680, 420), (1000, 530)])
@pytest.mark.parametrize("mode,metric", [(1, 1), (0, 0)])
def test_paper_resolutions(W, H, mode, metric):
    """Every source size of PAPER.md Table 1 -> 50x50: large bands run
    with fewer worker groups (ds_plan), unaligned rows (1170*3 = 3510 B) through the
    generic path; small frames, scores and dispositions bit-exact."""
    nsm = ns()
    n = 10
    sc, fr = scene_frames(W, H, n, seed=7, prevalence=0.95)
    small_o = O.downsample(hw3(fr, W, H), 50, 50)
    lr = sg.lr_weights(10, 4)
    ref = O.downsample(sg.background(sc.spec)[None], 50, 50)[0]
    s_tmp, _ = O.diff_detect(small_o, O.DDConfig(mode=mode, metric=metric, grid=10, t_diff_frames=3,
                                                 delta_diff=0.0, ref_image=ref, lr_w=lr[0], lr_b=lr[1]))
    fin = s_tmp[np.isfinite(s_tmp)]
    delta = float(np.quantile(fin, 0.5))
    ocfg, g = dd_pair(nsm, mode, metric, k=3, delta=delta, ref=ref, lr=lr)
    s_o, d_o = O.diff_detect(small_o, ocfg)
    res = _run(nsm, g, fr, W, H)
    _compare(res, small_o, s_o, d_o)


def test_ssd_overflow_shapes_rejected():
    """u32 SSDs: out_w*out_h*3*255^2 must stay below 2^32 (53 x 720 would wrap)."""
    nsm = ns()
    sc, fr = scene_frames(1280, 720, 2, seed=1)
    g = nsm.DD(mode=1, metric=0, out_w=53, out_h=720, t_diff_frames=1, delta_diff=0.0)
    with pytest.raises(nsm.NoScopeError):
        nsm.noscope_diff_detect(g, torch.from_numpy(fr).cuda(), 1280, 720)
    g = nsm.DD(mode=1, metric=0, out_w=53, out_h=415, t_diff_frames=1, delta_diff=0.0)   # 53*415*3*65025 < 2^32
    out = nsm.noscope_diff_detect(g, torch.from_numpy(fr).cuda(), 1280, 720)
    torch.cuda.synchronize()
    small_o = O.downsample(hw3(fr, 1280, 720), 415, 53)
    assert np.array_equal(out["small"].cpu().numpy()[:, :53 * 415 * 3], small_o.reshape(2, -1))
