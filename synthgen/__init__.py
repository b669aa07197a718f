"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is the ONLY code both sides may use (task rule ③).  It holds no
arithmetic of NoScope's method: it draws fixed-angle-camera video (static
textured background, per-frame sensor noise, moving bright rectangles), the
ground-truth labels the stand-in reference labeller returns, random-init CNN /
LR weights, threshold candidate grids and sweep records.  Everything is a
pure function of integer seeds through a counter-based hash (splitmix64), so
a CUDA renderer (``synthgen/synth_gpu.cu``) reproduces the frames byte for
byte without sharing code with the oracle.

Scene recipe (SURVEY.md §8(d) "Synthetic video"):
fixed-angle webcams; SPEC.md SynthSpec
 "axis-aligned bright rectangles on a darker background";
label = 1 iff a rectangle overlaps the frame.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from .hashing import (MIX, TAG_BG, TAG_NOISE, hash_key_np, splitmix64_np)
from .weights import (ARCH_GRID, PAPER_GRID, CnnArch, bf16_bits_to_f32, bf16_round_f32,
                      he_normal_weights, zero_weights)

__all__ = [
    "SceneSpec", "Scene", "make_scene", "render_frames", "render_frame",
    "frame_pitch", "CnnArch", "ARCH_GRID", "PAPER_GRID", "he_normal_weights",
    "bf16_round_f32", "bf16_bits_to_f32", "zero_weights", "background", "lr_weights", "logit_grid",
    "delta_grid", "random_sweep_records", "hash_key_np", "splitmix64_np",
    "MIX", "TAG_BG", "TAG_NOISE",
]

MAX_ACTIVE = 3  # "1-3 concurrent" rectangles


@dataclasses.dataclass(frozen=True)
class SceneSpec:
    """One synthetic fixed-angle camera stream."""
    width: int
    height: int
    n_frames: int
    seed: int
    stream: int = 0
    noise_sigma: int = 2          # integer sensor noise in [-sigma, sigma]
    prevalence: float = 0.15      # target fraction of frames with an object
    min_side_frac: float = 0.08   # rectangle side 8-20% of the frame side
    max_side_frac: float = 0.20
    min_speed: int = 1            # integer px/frame at source resolution
    max_speed: int = 4


@dataclasses.dataclass
class Scene:
    """A stream's event schedule, per-frame active slots and truth labels.

    events: int32 [E, 10] rows = (t0, t1, x0, y0, vx, vy, w, h, rgb, pad)
       where rectangle top-left at frame t is (x0 + vx*(t-t0), y0 + vy*(t-t0))
       and rgb packs the three channel values (r | g<<8 | b<<16).
    active: int32 [T, 3] event ids drawn in slot order (later slot on top),
       -1 = empty slot.
    truth: uint8 [T] ground-truth label (1 iff any rectangle overlaps).
    """
    spec: SceneSpec
    events: np.ndarray
    active: np.ndarray
    truth: np.ndarray


def frame_pitch(width: int, height: int) -> int:
    """Bytes between frames: W*H*3 rounded up to a 16-byte multiple.

    (The ABI's frame_pitch contract, include/noscope.h.)"""
    return (width * height * 3 + 15) // 16 * 16


def make_scene(spec: SceneSpec) -> Scene:
    """Draw the object schedule (Poisson arrivals, edge entries)."""
    W, H, T = spec.width, spec.height, spec.n_frames
    rng = np.random.Generator(np.random.PCG64([spec.seed, spec.stream, 7]))
    min_w = max(2, int(round(spec.min_side_frac * W)))
    max_w = max(min_w, int(round(spec.max_side_frac * W)))
    min_h = max(2, int(round(spec.min_side_frac * H)))
    max_h = max(min_h, int(round(spec.max_side_frac * H)))
    speeds = np.arange(spec.min_speed, spec.max_speed + 1)
    inv_speed = float(np.mean(1.0 / speeds))
    mean_dur = 0.5 * ((W + 0.5 * (min_w + max_w)) + (H + 0.5 * (min_h + max_h))) * inv_speed
    lam = -math.log(1.0 - spec.prevalence) / mean_dur if spec.prevalence > 0 else 0.0

    events = []
    active = np.full((T, MAX_ACTIVE), -1, dtype=np.int32)
    t = 0
    if lam > 0:
        t = int(rng.geometric(min(1.0, lam))) - 1
    while lam > 0 and t < T:
        w = int(rng.integers(min_w, max_w + 1))
        h = int(rng.integers(min_h, max_h + 1))
        v = int(rng.choice(speeds))
        edge = int(rng.integers(0, 4))  # 0 left, 1 right, 2 top, 3 bottom
        if edge == 0:
            x0, y0, vx, vy = 1 - w, int(rng.integers(0, H - h + 1)), v, 0
            dur = (W - 1 - x0) // v + 1
        elif edge == 1:
            x0, y0, vx, vy = W - 1, int(rng.integers(0, H - h + 1)), -v, 0
            dur = (x0 + w - 1) // v + 1
        elif edge == 2:
            x0, y0, vx, vy = int(rng.integers(0, W - w + 1)), 1 - h, 0, v
            dur = (H - 1 - y0) // v + 1
        else:
            x0, y0, vx, vy = int(rng.integers(0, W - w + 1)), H - 1, 0, -v
            dur = (y0 + h - 1) // v + 1
        rgb = [int(c) for c in rng.integers(200, 256, size=3)]
        t1 = min(T, t + dur)
        # place in the first slot free over the whole lifetime, else drop
        eid = len(events)
        for s in range(MAX_ACTIVE):
            if np.all(active[t:t1, s] < 0):
                active[t:t1, s] = eid
                events.append((t, t1, x0, y0, vx, vy, w, h,
                               rgb[0] | (rgb[1] << 8) | (rgb[2] << 16), 0))
                break
        t += int(rng.geometric(min(1.0, lam)))
    ev = np.array(events, dtype=np.int32).reshape(-1, 10)
    truth = (active >= 0).any(axis=1).astype(np.uint8)
    return Scene(spec, ev, active, truth)


def _background(spec: SceneSpec) -> np.ndarray:
    """Static texture, integer values in [40, 140] ("darker background")."""
    H, W = spec.height, spec.width
    yy, xx = np.meshgrid(np.arange(H, dtype=np.uint64), np.arange(W, dtype=np.uint64),
                         indexing="ij")
    h = hash_key_np(spec.seed, spec.stream, TAG_BG, yy, xx)
    out = np.empty((H, W, 3), dtype=np.int32)
    for c in range(3):
        out[..., c] = 40 + (((h >> np.uint64(16 * c)) & np.uint64(0xFFFF)) % np.uint64(101)).astype(np.int32)
    return out


def background(spec: SceneSpec) -> np.ndarray:
    """Noiseless, object-free background (the ideal reference image)."""
    return _background(spec).astype(np.uint8)


def render_frame(scene: Scene, t: int, bg: np.ndarray | None = None) -> np.ndarray:
    """uint8 [H, W, 3] frame t of the stream (random access by counter)."""
    spec = scene.spec
    H, W = spec.height, spec.width
    base = (_background(spec) if bg is None else bg.astype(np.int32)).copy()
    for s in range(MAX_ACTIVE):
        e = int(scene.active[t, s])
        if e < 0:
            continue
        t0, _, x0, y0, vx, vy, w, h, rgb, _ = (int(v) for v in scene.events[e])
        x = x0 + vx * (t - t0)
        y = y0 + vy * (t - t0)
        xa, xb = max(0, x), min(W, x + w)
        ya, yb = max(0, y), min(H, y + h)
        if xa < xb and ya < yb:
            for c in range(3):
                base[ya:yb, xa:xb, c] = (rgb >> (8 * c)) & 0xFF
    if spec.noise_sigma > 0:
        yy, xx = np.meshgrid(np.arange(H, dtype=np.uint64), np.arange(W, dtype=np.uint64),
                             indexing="ij")
        hn = hash_key_np(spec.seed, spec.stream, TAG_NOISE + np.uint64(t), yy, xx)
        span = np.uint64(2 * spec.noise_sigma + 1)
        for c in range(3):
            n = (((hn >> np.uint64(16 * c)) & np.uint64(0xFFFF)) % span).astype(np.int32) - spec.noise_sigma
            base[..., c] += n
    return np.clip(base, 0, 255).astype(np.uint8)


def render_frames(scene: Scene, t_begin: int = 0, t_end: int | None = None,
                  pitch: int | None = None) -> np.ndarray:
    """uint8 [n, pitch] frames t_begin..t_end-1, each padded to the frame pitch."""
    spec = scene.spec
    t_end = spec.n_frames if t_end is None else t_end
    pitch = frame_pitch(spec.width, spec.height) if pitch is None else pitch
    nb = spec.width * spec.height * 3
    out = np.zeros((t_end - t_begin, pitch), dtype=np.uint8)
    bg = _background(spec)
    for i, t in enumerate(range(t_begin, t_end)):
        out[i, :nb] = render_frame(scene, t, bg).reshape(-1)
    return out


def lr_weights(grid: int, seed: int) -> tuple[np.ndarray, np.float32]:
    """Blocked-DD logistic weights w_k ~ U[0,1] (float32), bias -4."""
    rng = np.random.Generator(np.random.PCG64([seed, 31]))
    w = rng.random(grid * grid).astype(np.float32)
    return w, np.float32(-4.0)


def delta_grid(scores: np.ndarray, n: int = 100) -> np.ndarray:
    """Strictly ascending float64 δ candidates: sentinels + log-spaced over the
    observed finite scores.  Input grid only."""
    s = scores[np.isfinite(scores)]
    lo = float(np.min(s)) if s.size else 0.0
    hi = float(np.max(s)) if s.size else 1.0
    inner = n - 2
    if hi - lo <= 0:
        mid = np.linspace(lo - 1.0, hi + 1.0, inner)
    else:
        shift = 1.0 - lo
        mid = np.exp(np.linspace(np.log(lo + shift), np.log(hi + shift), inner)) - shift
    g = np.concatenate([[-np.inf], mid, [np.inf]])
    g = np.unique(g.astype(np.float64))
    return g


def logit_grid(m: int = 100, lo: float = -8.0, hi: float = 8.0) -> np.ndarray:
    """Strictly ascending float32 logit candidates incl. ±inf."""
    mid = np.linspace(lo, hi, m - 2, dtype=np.float64).astype(np.float32)
    g = np.concatenate([[-np.inf], mid, [np.inf]]).astype(np.float32)
    return np.unique(g)


def random_sweep_records(n: int, seed: int, tie_frac: float = 0.2,
                         n_delta: int = 12, m: int = 10):
    """Random sweep instance with ties, ±inf scores and exact candidate hits.

    Returns (s f64[n], z f32[n], y u8[n], a u8[n], delta f64[nδ], u f32[m])."""
    rng = np.random.Generator(np.random.PCG64([seed, 53]))
    delta = np.unique(np.round(rng.normal(0, 2, n_delta), 1)).astype(np.float64)
    u = np.unique(np.round(rng.normal(0, 2, m), 1).astype(np.float32))
    if rng.random() < 0.5:
        u = np.unique(np.concatenate([u, np.float32([-np.inf])]))
    if rng.random() < 0.5:
        u = np.unique(np.concatenate([u, np.float32([np.inf])]))
    s = np.round(rng.normal(0, 2, n), 1)
    hit = rng.random(n) < tie_frac
    s[hit] = rng.choice(delta, size=int(hit.sum()))
    s[rng.random(n) < 0.1] = -np.inf
    s[rng.random(n) < 0.05] = np.inf
    z = np.round(rng.normal(0, 2, n), 1).astype(np.float32)
    hit = rng.random(n) < tie_frac
    z[hit] = rng.choice(u, size=int(hit.sum()))
    z[~np.isfinite(z)] = 0.0
    y = (rng.random(n) < 0.3).astype(np.uint8)
    a = (rng.random(n) < 0.2).astype(np.uint8)
    return s.astype(np.float64), z, y, a, delta, u
