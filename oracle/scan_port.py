"""The reference's CPU scan path restated — oracle / CPU-baseline only.

Restates ``scanattn.engine.scan_forward`` (engine.py:385-427) for timing the
reference's own CPU algorithm beside the GPU kernel (bench.py ``cpu_baseline``
and ``--impl reference``) and as a second FP32 comparator in tests:
  * per (b, h, query-tile) task, leaves (s, 1, v) with s = (Q_t K^T) * scale
    from one BLAS matmul per tile (engine.py:352-358);
  * level-synchronous doubling (Hillis–Steele) scan inside each B-key block,
    lane i combining with lane i - 2^l, tail block scanned at its own length
    (engine.py:148-176, 315-339);
  * block totals padded with the identity to a power of two and reduced by a
    pairwise up-sweep (engine.py:179-199, 364-371);
  * normalizer check and Y = W / S (engine.py:375-382);
  * tasks mapped over a thread pool; numpy releases the GIL inside its
    kernels, and the reduction tree depends only on (n, B), so the output is
    independent of the worker count (engine.py:11-13).
The combine is ``oracle.monoid.merge_lanes`` (monoid.py:160-200). Output is
bit-identical to the reference's FP32 scan (pinned by tests/golden).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .monoid import merge_lanes

__all__ = ["scan_forward_port", "tile_forward"]


def _doubling_last(m, S, W):
    """Inclusive doubling scan along axis 2 of (T, G, L) lanes; returns the
    last lane (the block totals), shapes (T, G) and (T, G, d_v)."""
    L = m.shape[2]
    step = 1
    while step < L:
        nm, nS, nW = merge_lanes(m[:, :, :-step], S[:, :, :-step], W[:, :, :-step],
                                 m[:, :, step:], S[:, :, step:], W[:, :, step:])
        m = np.concatenate([m[:, :, :step], nm], axis=2)
        S = np.concatenate([S[:, :, :step], nS], axis=2)
        W = np.concatenate([W[:, :, :step], nW], axis=2)
        step *= 2
    return m[:, :, -1], S[:, :, -1], W[:, :, -1]


def _upsweep_root(m, S, W):
    """Pairwise up-sweep over axis 1 (power-of-two lanes); returns the root."""
    K = m.shape[1]
    span = 1
    while span < K:
        left = slice(span - 1, K, 2 * span)
        right = slice(2 * span - 1, K, 2 * span)
        nm, nS, nW = merge_lanes(m[:, left], S[:, left], W[:, left],
                                 m[:, right], S[:, right], W[:, right])
        m[:, right], S[:, right], W[:, right] = nm, nS, nW
        span *= 2
    return S[:, K - 1], W[:, K - 1]


def tile_forward(Qt, K, V, scale, block_size):
    """One query tile against all keys (engine.py:342-382)."""
    T = Qt.shape[0]
    n, d_v = V.shape
    dt = Qt.dtype
    logits = np.empty((T, n), dtype=dt)
    np.matmul(Qt, K.T, out=logits)
    np.multiply(logits, dt.type(scale), out=logits)
    ones = np.ones((T, n), dtype=dt)
    vals = np.broadcast_to(V[None], (T, n, d_v))
    full, rem = divmod(n, block_size)
    tm, tS, tW = [], [], []
    for start, count, length in ((0, full, block_size), (full * block_size, 1, rem)):
        if count == 0 or length == 0:
            continue
        sl = slice(start, start + count * length)
        bm, bS, bW = _doubling_last(logits[:, sl].reshape(T, count, length),
                                    ones[:, sl].reshape(T, count, length),
                                    vals[:, sl].reshape(T, count, length, d_v))
        tm.append(bm)
        tS.append(bS)
        tW.append(bW)
    tm = np.concatenate(tm, axis=1)
    tS = np.concatenate(tS, axis=1)
    tW = np.concatenate(tW, axis=1)
    nb = tm.shape[1]
    padded = 1 << (0 if nb <= 1 else math.ceil(math.log2(nb)))
    pm = np.full((T, padded), -np.inf, dtype=dt)
    pS = np.zeros((T, padded), dtype=dt)
    pW = np.zeros((T, padded, d_v), dtype=dt)
    pm[:, :nb], pS[:, :nb], pW[:, :nb] = tm, tS, tW
    rS, rW = _upsweep_root(pm, pS, pW)
    if not np.all(np.isfinite(rS)) or np.any(rS <= 0):
        raise ArithmeticError("scan normalizer is zero or non-finite")
    return rW / rS[:, None]


def scan_forward_port(Q, K, V, scale=None, block_size=128, tile_q=64, workers=1,
                      dtype=np.float32, tiles=None):
    """Blocked-scan attention over every (b, h, query tile).

    ``tiles`` optionally restricts the work to a list of (b, h, q0) task
    starts (the bench's bounded CPU sample); the returned Y then only has
    those rows filled.
    """
    dt = np.dtype(dtype)
    Q, K, V = (np.asarray(x).astype(dt, copy=False) for x in (Q, K, V))
    b, h, n, d = Q.shape
    d_v = V.shape[3]
    sc = (1.0 / float(np.sqrt(d))) if scale is None else float(scale)
    Y = np.zeros((b, h, n, d_v), dtype=dt)
    if tiles is None:
        tiles = [(bi, hi, q0) for bi in range(b) for hi in range(h) for q0 in range(0, n, tile_q)]

    def run(task):
        bi, hi, q0 = task
        q1 = min(q0 + tile_q, n)
        Y[bi, hi, q0:q1] = tile_forward(Q[bi, hi, q0:q1], K[bi, hi], V[bi, hi], sc, block_size)

    if workers == "auto":
        workers = os.cpu_count() or 1
    if workers == 1 or len(tiles) == 1:
        for t in tiles:
            run(t)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(run, tiles))
    return Y
