"""GPU parity of the evaluation harness: noscope_eval_labels
counts bit-exact vs the oracle, and the factor-analysis / lesion rows of the GPU
cascade identical to the oracle's (accuracy, FP, FN, stage counts, modeled
speedup).  Route thresholds sit in gaps of the oracle's logits wider than the
CNN parity bound."""
import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import hw3, ns, requires_gpu, scene_frames

pytestmark = [pytest.mark.gpu, requires_gpu]


@pytest.mark.parametrize("n,shift", [(29, 0), (30, 0), (95, 0), (480, 0), (100_003, 0), (4_800_007, 0),
                                     (100_003, 1)])
def test_eval_labels_counts(n, shift):
    """30-frame windows take the 16-byte-vector kernel (480-frame blocks + a generic tail)
    when both tracks are 16-byte aligned (shift = 0), the generic kernel otherwise."""
    nsm = ns()
    rng = np.random.default_rng(n)
    ref = (rng.random(n) < 0.3).astype(np.uint8)
    pred = ref.copy()
    flip = rng.random(n) < 0.04
    pred[flip] ^= 1
    pred[pred == 1] = rng.integers(1, 255, int((pred == 1).sum()))       # any nonzero = present
    pd = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
    rd = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
    pd[shift:shift + n] = torch.from_numpy(pred).cuda()
    rd[shift:shift + n] = torch.from_numpy(ref).cuda()
    ev = nsm.noscope_eval_labels(pd[shift:shift + n], rd[shift:shift + n])
    fp, fn, tp, tn = O.fp_fn(pred, ref)
    assert (ev["fp"], ev["fn"], ev["tp"], ev["tn"]) == (fp, fn, tp, tn)
    assert ev["windows"] == n // 30
    if n >= 30:
        assert ev["correct_windows"] / ev["windows"] == O.windowed_accuracy(pred, ref)


@pytest.mark.parametrize("rows", ["factor", "lesion"])
def test_factor_analysis_matches_oracle(rows):
    nsm = ns()
    from paper_1703_02529_b200 import harness as H
    from synthgen.gpu import GpuScene, truth_labeller_address
    n = 240
    sc, fr = scene_frames(50, 50, n, seed=41, prevalence=0.35)
    small = hw3(fr, 50, 50)
    y = sc.truth[:n].astype(np.uint8)
    ref = sg.background(sc.spec)
    arch = sg.CnnArch(2, 32, 32)
    w = sg.he_normal_weights(arch, 5)
    z_o = O.cnn_logits(small, arch, w).astype(np.float64)
    zs = np.sort(z_o)
    mid = np.arange(len(zs) // 10, len(zs) - len(zs) // 10)
    gaps = zs[mid + 1] - zs[mid]
    two = mid[np.argsort(gaps)[-2:]]                     # the two widest interior gaps
    lo, hi = sorted(float(np.float32(0.5 * (zs[i] + zs[i + 1]))) for i in two)
    margin = min(min(abs(z_o - lo)), min(abs(z_o - hi)))
    z_g = nsm.noscope_specialized_infer(nsm.Arch(2, 32, 32), nsm.Weights(w),
                                        torch.from_numpy(np.ascontiguousarray(
                                            np.pad(fr[:, :7500], ((0, 0), (0, 4))))).cuda())
    dz = np.abs(z_g.cpu().numpy() - z_o).max()
    assert margin > dz, (margin, dz)                      # no frame can change route
    timing = (2, 30, 1000)
    ocfg = O.DDConfig(mode=0, metric=0, t_skip_frames=3, delta_diff=15.0, ref_image=ref)
    orows = O.factor_analysis(small, ocfg, arch, w, lo, hi, y, timing,
                              rows=O.FACTOR_ROWS if rows == "factor" else O.LESION_ROWS)
    dd = nsm.DD(mode=0, metric=0, t_skip_frames=3, delta_diff=15.0, ref_image=torch.from_numpy(ref).cuda())
    gs = GpuScene(sc)
    grows = H.factor_analysis(torch.from_numpy(fr).cuda(), 50, 50, dd, nsm.Arch(2, 32, 32), nsm.Weights(w),
                              lo, hi, truth_labeller_address(), gs.truth, torch.from_numpy(y).cuda(), timing,
                              rows=H.FACTOR_ROWS if rows == "factor" else H.LESION_ROWS)
    for o, g in zip(orows, grows):
        assert o == g, (o, g)
