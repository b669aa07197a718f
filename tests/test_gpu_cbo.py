"""GPU parity of the full CBO search (reading R-23) against
the oracle's cbo_search: the same (DD config, CNN, delta_j, c_low_l, c_high_h)
and the same integer cost / FP / FN / U.  Logit candidates sit in gaps of the
oracle's logits wider than the CNN parity bound, so the bf16 CNN cannot move a
frame across a candidate."""
import numpy as np
import pytest
import torch

import oracle as O
import synthgen as sg
from gpu_util import hw3, ns, requires_gpu, scene_frames

pytestmark = [pytest.mark.gpu, requires_gpu]


def _gap_candidates(zs, margin, k):
    z = np.sort(np.concatenate(zs).astype(np.float64))
    mids = [(0.5 * (a + b), b - a) for a, b in zip(z[:-1], z[1:]) if b - a > 2 * margin]
    mids.sort()
    pick = [mids[int(i)][0] for i in np.linspace(0, len(mids) - 1, min(k, len(mids)))]
    return np.array([-np.inf] + sorted(set(pick)) + [np.inf], np.float32)


@pytest.mark.parametrize("limits,skip_first,src", [((8, 8), False, 50), ((0, 0), False, 50),
                                                  ((8, 8), True, 50), ((8, 8), True, 100)])
def test_cbo_search_matches_oracle(limits, skip_first, src):
    """skip_first: the t_skip = 2 DD config comes first, so the CNN input cannot be
    the first DD pass's small frames (that pass downsamples only checked frames and
    anchors); src = 100: the band-pipeline downsample (100x100 -> 50x50)."""
    nsm = ns()
    n = 400
    sc, fr = scene_frames(src, src, n, seed=31, prevalence=0.35)
    small = O.downsample(hw3(fr, src, src), 50, 50)
    y = sc.truth[:n].astype(np.uint8)
    ref = O.downsample(sg.background(sc.spec)[None], 50, 50)[0]
    lr_w = np.full(25, 0.02, np.float32)
    ocfgs = [O.DDConfig(mode=0, metric=0, delta_diff=0.0, ref_image=ref),
             O.DDConfig(mode=1, metric=1, grid=5, t_diff_frames=5, t_skip_frames=2, delta_diff=0.0,
                        lr_w=lr_w, lr_b=-1.0)]
    if skip_first:
        ocfgs = ocfgs[::-1]
    grids = [sg.delta_grid(O.diff_detect(small, c)[0], 12) for c in ocfgs]
    arch = sg.CnnArch(2, 32, 32)
    ws = [sg.he_normal_weights(arch, 3), sg.he_normal_weights(arch, 9)]
    z_o = [O.cnn_logits(small, arch, w) for w in ws]
    u = _gap_candidates(z_o, 0.03, 14)
    t_snn = [40, 25]
    fp, fn = limits
    d_o, c_o, b_o = O.cbo_search(small, y, ocfgs, grids, [(arch, w, t) for w, t in zip(ws, t_snn)], u,
                                 5, 1000, fp, fn)
    dev = "cuda"
    gi = [1, 0] if skip_first else [0, 1]
    dds = [(nsm.DD(mode=0, metric=0, delta_diff=0.0, ref_image=torch.from_numpy(ref).to(dev)),
            torch.from_numpy(grids[gi[0]]).to(dev)),
           (nsm.DD(mode=1, metric=1, grid=5, t_diff_frames=5, t_skip_frames=2, delta_diff=0.0,
                   lr_weights=torch.from_numpy(lr_w).to(dev), lr_bias=-1.0), torch.from_numpy(grids[gi[1]]).to(dev))]
    if skip_first:
        dds = dds[::-1]
    A = nsm.Arch(2, 32, 32)
    cnns = [(A, nsm.Weights(w), t) for w, t in zip(ws, t_snn)]
    frames = torch.from_numpy(fr).to(dev)
    d, c, b, code = nsm.noscope_cbo_search(dds, cnns, frames, src, src, torch.from_numpy(y).to(dev),
                                           torch.from_numpy(u).to(dev), 5, 1000, fp, fn)
    assert (d, c) == (d_o, c_o)
    assert (b["j"], b["l"], b["h"]) == (b_o["j"], b_o["l"], b_o["h"])
    assert (b["cost_ps"], b["fp"], b["fn"], b["uncertain"], b["fired"]) == \
        (b_o["cost"], b_o["fp"], b_o["fn"], b_o["U"], b_o["F"])
    assert bool(b["feasible"]) == bool(b_o["feasible"]) and (code == 0) == bool(b_o["feasible"])
