"""Seeded problem generation and the depth bound, restated — oracle only.

Follows /root/reference/pkg/src/scanattn:
  * scan_depth / depth_cap: engine.py:43-60
    L(n, B) = ceil(log2 min(B, n)) + 2 ceil(log2 ceil(n / B)) + 3
  * SCENARIOS presets: tensorio.py:118-122
  * generate: tensorio.py:125-195 — one Philox stream per (tensor, b, h) slab
    keyed [seed, (tag << 48) | (b << 24) | h] with tags Q=1, K=2, V=3
    (tensorio.py:167-174); N(0,1) drawn in float64, multiplied by the
    scenario's power-of-two feature scale, then cast to the target dtype.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["SCENARIOS", "scan_depth", "depth_cap", "generate", "slab"]

SCENARIOS = {
    "regular": dict(b=2, h=4, n=256, d=32, d_v=32, feature_scale=1.0),
    "long": dict(b=1, h=1, n=4096, d=32, d_v=32, feature_scale=1.0),
    "stress": dict(b=2, h=2, n=1024, d=32, d_v=32, feature_scale=8.0),
}

_TAG = {"Q": 1, "K": 2, "V": 3}


def _clog2(x):
    return 0 if x <= 1 else int(math.ceil(math.log2(x)))


def scan_depth(n, block_size=128):
    if n < 1 or block_size < 1:
        raise ValueError("n and block_size must be >= 1")
    blocks = -(-n // block_size)
    return _clog2(min(block_size, n)) + 2 * _clog2(blocks) + 3


def depth_cap(n):
    return 2 * _clog2(n) + 3


def slab(seed, tensor, b_idx, h_idx, rows, width, feature_scale=1.0):
    """float64 N(0,1) slab for one (tensor, b, h) — tensorio.py:170-174, 188-193."""
    key = [np.uint64(seed), np.uint64((_TAG[tensor] << 48) | (b_idx << 24) | h_idx)]
    x = np.random.Generator(np.random.Philox(key=key)).standard_normal((rows, width))
    if feature_scale != 1.0:
        x *= feature_scale
    return x


def generate(seed, scenario="regular", b=1, h=1, n=128, d=32, d_v=32, dtype=np.float64):
    """Return (Q, K, V) numpy arrays of shape (b, h, n, d|d_v) in ``dtype``."""
    if scenario not in SCENARIOS:
        raise ValueError(f"unknown scenario {scenario!r}")
    fs = SCENARIOS[scenario]["feature_scale"]
    dt = np.dtype(dtype)
    out = []
    for name, width in (("Q", d), ("K", d), ("V", d_v)):
        arr = np.empty((b, h, n, width), dtype=dt)
        for bi in range(b):
            for hi in range(h):
                arr[bi, hi] = slab(seed, name, bi, hi, n, width, fs).astype(dt)
        out.append(arr)
    return tuple(out)
