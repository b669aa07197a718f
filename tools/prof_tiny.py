"""The tiny config (BASELINE configs[0]) cascade a few times, for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
print(bench.tiny_config(torch.device("cuda", 0)))
