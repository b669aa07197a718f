"""Counter-based hash (splitmix64) used by the synthetic generators.

The CUDA renderer in synthgen/synth_gpu.cu implements the same chain; the
test tests/test_synthgen.py checks the two byte for byte."""
from __future__ import annotations

import numpy as np

MIX = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
TAG_BG = np.uint64(1)
TAG_NOISE = np.uint64(1 << 32)


def splitmix64_np(x):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + MIX
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def hash_key_np(seed, stream, tag, y, x):
    """h = sm(sm(sm(sm(sm(seed) ^ stream) ^ tag) ^ y) ^ x)."""
    k = splitmix64_np(np.uint64(seed))
    k = splitmix64_np(k ^ np.uint64(stream))
    k = splitmix64_np(k ^ np.uint64(tag))
    k = splitmix64_np(k ^ np.asarray(y, dtype=np.uint64))
    return splitmix64_np(k ^ np.asarray(x, dtype=np.uint64))
