"""Block totals, the two-pass inter-block combine and exclusive block
prefixes, restated in numpy — oracle only.

Follows /root/reference/pkg/src/scanattn/engine.py:
  * _upsweep (engine.py:179-199): identity-padded power-of-two lane array,
    level l merges lane (half-1 + k*stride) INTO lane (stride-1 + k*stride)
    as ``left (+) right``; the grand total lands in the last lane;
  * _downsweep (engine.py:202-231): the root is reset to the identity; per
    level (top down) the left lane takes the right lane's running prefix and
    the right lane becomes ``prefix (+) old_left``;
  * inter_block_combine (engine.py:265-297): up-sweep total, optional
    exclusive prefixes (identity first);
  * blockwise_states (engine.py:430-451) — here through the FP64 partial
    state of each key block (the reference computes each block with its
    intra-block doubling scan in the configured precision; the two agree to
    rounding).

Vectorised over a leading row axis: m, S are (rows, K), W is (rows, K, d_v).
"""

from __future__ import annotations

import numpy as np

from .attention import partial_state_fp64
from .monoid import merge_lanes

__all__ = ["upsweep", "downsweep", "inter_block_combine", "blockwise_states_fp64"]


def _clog2(x):
    return 0 if x <= 1 else int(np.ceil(np.log2(x)))


def _pad(m, S, W):
    m, S, W = np.asarray(m), np.asarray(S), np.asarray(W)
    rows, K = m.shape
    K_pad = 1 << _clog2(K)
    tm = np.full((rows, K_pad), -np.inf, dtype=m.dtype)
    tS = np.zeros((rows, K_pad), dtype=m.dtype)
    tW = np.zeros((rows, K_pad, W.shape[2]), dtype=m.dtype)
    tm[:, :K], tS[:, :K], tW[:, :K] = m, S, W
    return tm, tS, tW


def upsweep(tm, tS, tW):
    """In place (engine.py:179-199)."""
    K_pad = tm.shape[1]
    for lvl in range(_clog2(K_pad)):
        stride, half = 2 << lvl, 1 << lvl
        left = slice(half - 1, K_pad, stride)
        right = slice(stride - 1, K_pad, stride)
        mm, SS, WW = merge_lanes(tm[:, left], tS[:, left], tW[:, left],
                                 tm[:, right], tS[:, right], tW[:, right])
        tm[:, right], tS[:, right], tW[:, right] = mm, SS, WW


def downsweep(tm, tS, tW):
    """In place (engine.py:202-231)."""
    K_pad = tm.shape[1]
    tm[:, K_pad - 1] = -np.inf
    tS[:, K_pad - 1] = 0.0
    tW[:, K_pad - 1] = 0.0
    for lvl in reversed(range(_clog2(K_pad))):
        stride, half = 2 << lvl, 1 << lvl
        left = slice(half - 1, K_pad, stride)
        right = slice(stride - 1, K_pad, stride)
        lm, lS, lW = tm[:, left].copy(), tS[:, left].copy(), tW[:, left].copy()
        tm[:, left], tS[:, left], tW[:, left] = tm[:, right], tS[:, right], tW[:, right]
        mm, SS, WW = merge_lanes(tm[:, right], tS[:, right], tW[:, right], lm, lS, lW)
        tm[:, right], tS[:, right], tW[:, right] = mm, SS, WW


def inter_block_combine(m, S, W, return_prefixes=False):
    """(engine.py:265-297) -> total (m, S, W) per row [, exclusive prefixes
    (rows, K) / (rows, K, d_v)]."""
    K = np.asarray(m).shape[1]
    if K == 0:
        raise ValueError("no block totals to combine")
    tm, tS, tW = _pad(m, S, W)
    upsweep(tm, tS, tW)
    total = (tm[:, -1].copy(), tS[:, -1].copy(), tW[:, -1].copy())
    if not return_prefixes:
        return total
    downsweep(tm, tS, tW)
    return total, (tm[:, :K], tS[:, :K], tW[:, :K])


def blockwise_states_fp64(Q, K, V, block_size, scale=None):
    """FP64 (m, S, W) of every key block [j*B, min((j+1)*B, n_kv)) for every
    query row: m, S (b, h, n_q, nblocks), W (b, h, n_q, nblocks, d_v)."""
    n_kv = np.asarray(K).shape[2]
    nb = -(-n_kv // block_size)
    parts = [partial_state_fp64(Q, K, V, j * block_size, min((j + 1) * block_size, n_kv), scale)
             for j in range(nb)]
    m = np.stack([p[0] for p in parts], axis=-1)
    S = np.stack([p[1] for p in parts], axis=-1)
    W = np.stack([p[2] for p in parts], axis=-2)
    return m, S, W
