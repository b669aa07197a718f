"""The training path's tcgen05 GEMM (csrc/gemm_tc.cu, 3xTF32 on kind::tf32) against
numpy fp64 on ragged shapes, every operand orientation the backward pass uses,
and split-K.  Bar: fp32 accuracy — |C - C64| <= 2^-20 * sum_k |a_mk b_kn| + 1e-30
per element (a single-pass TF32 product would miss it by ~2^-11)."""
import numpy as np
import pytest
import torch

from gpu_util import ns, requires_gpu

pytestmark = [pytest.mark.gpu, requires_gpu]


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (130, 27, 27), (64, 32, 4608), (32, 27, 160000), (257, 300, 70),
                                   (1000, 1, 5000), (160000, 32, 27)])
@pytest.mark.parametrize("ta,tb", [(False, True), (True, False), (False, False)])
def test_tc_gemm_fp32_accuracy(M, N, K, ta, tb):
    nsm = ns()
    if M * K > 2e7 and ta:
        pytest.skip("covered by the untransposed case")
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    a = rng.normal(0, 1, (K, M) if ta else (M, K)).astype(np.float32)
    b = rng.normal(0, 1, (N, K) if tb else (K, N)).astype(np.float32)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    sam, sak = (1, M) if ta else (K, 1)
    sbn, sbk = (K, 1) if tb else (1, N)
    C = nsm.debug_tc_gemm(A, sam, sak, B, sbn, sbk, M, N, K).cpu().numpy()
    a64 = (a.T if ta else a).astype(np.float64)
    b64 = (b.T if tb else b).astype(np.float64)
    ref = a64 @ b64
    bound = np.abs(a64) @ np.abs(b64) * 2.0 ** -20 + 1e-30
    assert np.all(np.abs(C - ref) <= bound), float(np.max(np.abs(C - ref) / bound))
