"""One epoch of specialized-CNN training on 2,048 frames (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synthgen as sg  # noqa: E402
from paper_1703_02529_b200 import noscope as N  # noqa: E402
from synthgen.gpu import GpuScene  # noqa: E402
n = 2048 + 256
sc = sg.make_scene(sg.SceneSpec(50, 50, n, seed=3, prevalence=0.3))
gs = GpuScene(sc)
small = torch.empty((n, 7504), dtype=torch.uint8, device="cuda")
gs.render(small, 0, n)
arch = sg.CnnArch(2, 32, 32)
A = N.Arch(2, 32, 32)
p = N.params_from_weight_dict(A, sg.he_normal_weights(arch, 3))
perms = torch.randperm(2048, device="cuda").to(torch.int32).reshape(1, -1)
print(N.noscope_cnn_train(A, p, small, gs.truth[:n].contiguous(), perms,
                          torch.arange(2048, n, dtype=torch.int32, device="cuda"), batch=int(sys.argv[1]) if len(sys.argv) > 1 else 64))
