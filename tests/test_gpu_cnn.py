"""GPU parity: the tcgen05 specialized CNN (noscope_specialized_infer) against the
oracle's fp64 forward on the same bf16 weights and inputs.  Bar: |z_gpu - z_oracle|
<= 2e-2 absolute (north star).  Also checks the conv1 activation map directly
(layer-level parity) and gather-by-index / device-count semantics."""
import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import hw3, ns, requires_gpu, scene_frames

pytestmark = [pytest.mark.gpu, requires_gpu]
TOL = 2e-2


def _small(n, seed):
    sc, fr = scene_frames(50, 50, n, seed=seed, prevalence=0.6)
    pitch = 7504
    small = np.zeros((n, pitch), np.uint8)
    small[:, :7500] = fr[:, :7500]
    return small, hw3(fr, 50, 50)


@pytest.mark.parametrize("arch", sg.ARCH_GRID, ids=lambda a: a.name)
def test_cnn_logits_vs_oracle(arch):
    nsm = ns()
    n = 203                                             # several tiles + ragged tail
    small, g = _small(n, 11)
    w = sg.he_normal_weights(arch, 3)
    z_o = O.cnn_logits(g, arch, w)
    W = nsm.Weights(w)
    A = nsm.Arch(arch.n_conv, arch.base_filters, arch.dense)
    z = nsm.noscope_specialized_infer(A, W, torch.from_numpy(small).cuda())
    torch.cuda.synchronize()
    z = z.cpu().numpy()
    err = np.abs(z - z_o)
    assert err.max() <= TOL, (arch.name, err.max(), np.argmax(err))
    assert np.isfinite(z).all()


def _stacked_map(ws, lay, l, n):
    """Decode conv layer l's stacked input map (internal.h layout) for n frames:
    returns (interior [n, H, W, C] as float64, separator/guard rows as uint16)."""
    off, R, H, C = lay[4 * l: 4 * l + 4]
    Wq, P, G = H + 1, (H + 1) * (H + 1), H + 2
    planes = ws[off:off + (C // 8) * R * 16].cpu().numpy().view(np.uint16).reshape(C // 8, R, 8)
    body = planes[:, G:G + n * P, :].reshape(C // 8, n, H + 1, Wq, 8)
    inner = body[:, :, 1:, :H, :].transpose(1, 2, 3, 0, 4).reshape(n, H, H, C)
    inner = (inner.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    seps = np.concatenate([body[:, :, 0, :, :].ravel(), body[:, :, :, H, :].ravel(),
                           planes[:, :G, :].ravel(), planes[:, G + n * P:G + n * P + Wq, :].ravel()])
    return inner, seps


def _layer_check(got, ref):
    diff = np.abs(got - ref)
    # fp32 accumulation vs fp64: at most one bf16 ulp apart, except where the
    # sum cancels to near zero (fp32 sum error ~ K * 2^-24 * sum|w x| = O(1e-5))
    bad = ~(diff <= np.abs(ref) * 2 ** -7 + 2.0 ** -12)
    assert not bad.any(), (diff.max(), bad.sum(), np.argwhere(bad)[:5], got[bad][:5], ref[bad][:5])
    assert (diff == 0).mean() > 0.99, (diff == 0).mean()


def test_conv1_activation_map():
    """Layer-level parity of conv1 (base_filters = 64 materialises the conv1 map
    in the stacked layout; base_filters = 32 keeps it on chip) incl. the zero
    separators / guards that are the next conv's padding."""
    nsm = ns()
    arch = sg.CnnArch(2, 64, 32)
    n = 5
    small, g = _small(n, 12)
    w = sg.he_normal_weights(arch, 4)
    A = nsm.Arch(2, 64, 32)
    ws = nsm.workspace(nsm.OP_SPECIALIZED_INFER, None, A, n)
    ws.fill_(0x7F)                                     # stale bytes must not leak into the map
    nsm.noscope_specialized_infer(A, nsm.Weights(w), torch.from_numpy(small).cuda(), ws=ws)
    torch.cuda.synchronize()
    lay = nsm.debug_cnn_layout(A, n)
    got, seps = _stacked_map(ws, lay, 1, n)
    assert np.all(seps == 0)
    x = O.normalize_input(g, arch.chan_mean)
    a1 = O.conv3x3_same(x, O.bf16_bits_to_f64(w["conv_w"][0]), w["conv_b"][0].astype(np.float64))
    _layer_check(got, O.bf16_round(O.maxpool2x2_floor(np.maximum(a1, 0))))


@pytest.mark.parametrize("C", [32, 64])
def test_conv2_and_conv3_maps_L4(C):
    """Layer-level parity of the conv2 output (conv3 input) and the conv3 output
    (conv4 input) of the 4-layer networks: for C = 32 the conv2 map comes out of
    the fused conv1+conv2 kernel, for C = 64 out of the generic layer kernel."""
    nsm = ns()
    arch = sg.CnnArch(4, C, 32)
    n = 7
    small, g = _small(n, 15)
    w = sg.he_normal_weights(arch, 6)
    A = nsm.Arch(4, C, 32)
    ws = nsm.workspace(nsm.OP_SPECIALIZED_INFER, None, A, n)
    ws.fill_(0x7F)
    nsm.noscope_specialized_infer(A, nsm.Weights(w), torch.from_numpy(small).cuda(), ws=ws)
    torch.cuda.synchronize()
    lay = nsm.debug_cnn_layout(A, n)
    x = O.normalize_input(g, arch.chan_mean)
    checked = 0
    for l in range(3):
        a = O.conv3x3_same(x, O.bf16_bits_to_f64(w["conv_w"][l]), w["conv_b"][l].astype(np.float64))
        x = O.bf16_round(O.maxpool2x2_floor(np.maximum(a, 0)))
        if lay[4 * (l + 1)] >= 0:                        # layer l's output is materialised
            got, seps = _stacked_map(ws, lay, l + 1, n)
            assert np.all(seps == 0), l
            _layer_check(got, x)
            x = got          # continue from the GPU map so layer errors do not compound
            checked += 1
    assert checked == (3 if C == 64 else 2)


def test_cnn_gather_by_index_and_device_count():
    nsm = ns()
    arch = sg.CnnArch(2, 32, 32)
    small, g = _small(300, 13)
    w = sg.he_normal_weights(arch, 5)
    W = nsm.Weights(w)
    A = nsm.Arch(2, 32, 32)
    idx = np.array(sorted(np.random.default_rng(1).choice(300, 150, replace=False)), np.int32)
    cnt = torch.tensor([97], dtype=torch.int64, device="cuda")
    out = torch.full((150,), 12345.0, device="cuda")
    nsm.noscope_specialized_infer(A, W, torch.from_numpy(small).cuda(), idx=torch.from_numpy(idx).cuda(),
                                  n_dev=cnt, n_max=150, logits=out)
    torch.cuda.synchronize()
    z = out.cpu().numpy()
    z_o = O.cnn_logits(g[idx[:97]], arch, w)
    assert np.abs(z[:97] - z_o).max() <= TOL
    assert np.all(z[97:] == 12345.0)                      # beyond the device count: untouched


def test_cnn_zero_and_bias_weights():
    nsm = ns()
    arch = sg.CnnArch(4, 64, 128)
    w = sg.zero_weights(arch)
    w["fc2_b"] = np.float32([np.log(3.0)])
    small, _ = _small(20, 14)
    z = nsm.noscope_specialized_infer(nsm.Arch(4, 64, 128), nsm.Weights(w), torch.from_numpy(small).cuda())
    torch.cuda.synchronize()
    assert np.allclose(1 / (1 + np.exp(-z.cpu().numpy())), 0.75, atol=1e-6)


@pytest.mark.parametrize("L,C", [(2, 32), (2, 64), (4, 64), (4, 32), (2, 16), (4, 16)])
def test_cnn_multi_chunk_sampled(L, C):
    """More frames than one internal chunk: the layer kernels see
    chunk_base > 0 and a ragged last chunk.  Sampled frames from both chunks,
    including the chunk boundary, against the oracle."""
    nsm = ns()
    from synthgen.gpu import GpuScene
    chunk = nsm.debug_cnn_layout(nsm.Arch(L, C, 32), 1 << 20)[18]      # internal chunk size
    n = chunk + 301
    sc = sg.make_scene(sg.SceneSpec(50, 50, n, seed=19, prevalence=0.4))
    small = torch.empty((n, 7504), dtype=torch.uint8, device="cuda")   # rendered on device
    GpuScene(sc).render(small, 0, n)
    arch = sg.CnnArch(L, C, 32)
    w = sg.he_normal_weights(arch, 8)
    z = nsm.noscope_specialized_infer(nsm.Arch(L, C, 32), nsm.Weights(w), small)
    torch.cuda.synchronize()
    z = z.cpu().numpy()
    pick = np.array([0, 1, chunk // 2, chunk - 2, chunk - 1, chunk, chunk + 1, chunk + 108, n - 2, n - 1])
    bg = sg.background(sc.spec)
    g = np.stack([sg.render_frame(sc, int(t), bg) for t in pick])
    assert np.array_equal(small[torch.from_numpy(pick).cuda(), :7500].cpu().numpy(), g.reshape(len(pick), -1))
    z_o = O.cnn_logits(g, arch, w)
    assert np.abs(z[pick] - z_o).max() <= TOL
    assert np.isfinite(z).all()


@pytest.mark.parametrize("L,C,D", [(2, 32, 64), (2, 32, 256), (2, 64, 64), (4, 32, 256), (4, 64, 256)],
                         ids=lambda v: str(v))
def test_cnn_dense_64_and_256(L, C, D):
    """The paper's dense widths 64 and 256 (Table 2 picks D = 256 for
    amsterdam and elevator), beyond BASELINE's D in {32, 128}."""
    nsm = ns()
    n = 203
    small, g = _small(n, 12)
    arch = sg.CnnArch(L, C, D)
    w = sg.he_normal_weights(arch, 5)
    z_o = O.cnn_logits(g, arch, w)
    z = nsm.noscope_specialized_infer(nsm.Arch(L, C, D), nsm.Weights(w), torch.from_numpy(small).cuda())
    torch.cuda.synchronize()
    err = np.abs(z.cpu().numpy() - z_o)
    assert err.max() <= TOL, (arch.name, err.max())


def test_cnn_bench_batch_full_parity():
    """The bench's CNN at its in-cascade batch size: L2C32D32 on 16,384 frames (the
    webcam hour fires ~16.2k frames per call, ~110 per CTA, so every ring and phase
    of the fused kernel wraps many times), compared element-wise with the full
    oracle on every frame."""
    nsm = ns()
    n = 16384
    sc, fr = scene_frames(50, 50, n, seed=21, prevalence=0.5)
    small = np.zeros((n, 7504), np.uint8)
    small[:, :7500] = fr[:, :7500]
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 1)
    z = nsm.noscope_specialized_infer(nsm.Arch(2, 32, 32), nsm.Weights(w), torch.from_numpy(small).cuda())
    torch.cuda.synchronize()
    z = z.cpu().numpy()
    z_o = O.cnn_logits(hw3(fr, 50, 50), arch, w, batch=1024)
    err = np.abs(z - z_o)
    assert err.max() <= TOL, (err.max(), int(np.argmax(err)))
    assert np.isfinite(z).all()


@pytest.mark.parametrize("arch", [a for a in sg.PAPER_GRID if a.base_filters == 16], ids=lambda a: a.name)
def test_cnn_base_filters_16(arch):
    """C = 16 (Table 2's choice for coral and night-street): the paper's
    24-configuration grid = {2, 4} layers x {16, 32, 64} filters x
    {32, 64, 128, 256} dense; the C = 16 rows against the oracle."""
    nsm = ns()
    n = 203
    small, g = _small(n, 13)
    w = sg.he_normal_weights(arch, 6)
    z_o = O.cnn_logits(g, arch, w)
    A = nsm.Arch(arch.n_conv, arch.base_filters, arch.dense)
    z = nsm.noscope_specialized_infer(A, nsm.Weights(w), torch.from_numpy(small).cuda())
    torch.cuda.synchronize()
    err = np.abs(z.cpu().numpy() - z_o)
    assert err.max() <= TOL, (arch.name, err.max())
