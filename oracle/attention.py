"""FP64 attention references and the parity predicates — oracle only.

Follows /root/reference/pkg/src/scanattn:
  * naive_attention: oracles.py:74-104 — per (b, h) slice, scores = (Q K^T) *
    scale, subtract the row max, exp, row sums, Y = (P V) / s; the FP64 run is
    the ground truth of every parity test.
  * vectorized_oracle probabilities: oracles.py:107-122 (argmax checks).
  * bound_check threshold and per-row error: verify.py:320-358 —
    err_row = ||y - y64||_2 / max(||y64||_2, tiny), threshold =
    2^-24 * scan_depth(n, B) * slack with slack 8 (verify.py:49).
Additions for sizes the n x n matrix cannot reach (n >= 64K):
  * sampled_rows_fp64 restates oracles.py:92-98 for a chosen set of rows;
  * partial_state_fp64 is the (m, S, W) triple of a key range in FP64
    (the StateTriple of monoid.py:73-119 for that range, Proposition 1).
"""

from __future__ import annotations

import numpy as np

from .problems import scan_depth

__all__ = [
    "naive_attention",
    "vectorized_probs",
    "sampled_rows_fp64",
    "partial_state_fp64",
    "bound_threshold",
    "row_rel_err",
    "U32",
    "DEFAULT_SLACK",
]

U32 = 2.0 ** -24
DEFAULT_SLACK = 8.0


def _scale(d):
    return 1.0 / float(np.sqrt(d))


def naive_attention(Q, K, V, scale=None, dtype=np.float64, return_p=False):
    """Row-max-stabilised exact attention in ``dtype`` (oracles.py:74-104)."""
    dt = np.dtype(dtype)
    Q, K, V = (np.asarray(x).astype(dt, copy=False) for x in (Q, K, V))
    b, h, n_q, d = Q.shape
    d_v = V.shape[3]
    sc = dt.type(_scale(d) if scale is None else scale)
    Y = np.empty((b, h, n_q, d_v), dtype=dt)
    P = np.empty((b, h, n_q, K.shape[2]), dtype=dt) if return_p else None
    for bi in range(b):
        for hi in range(h):
            s = (Q[bi, hi] @ K[bi, hi].T) * sc
            m = s.max(axis=1, keepdims=True)
            np.subtract(s, m, out=s)
            np.exp(s, out=s)
            tot = s.sum(axis=1, keepdims=True)
            if not np.all(np.isfinite(tot)) or np.any(tot <= 0):
                raise ArithmeticError("softmax normalizer is zero or non-finite")
            Y[bi, hi] = (s @ V[bi, hi]) / tot
            if return_p:
                P[bi, hi] = s / tot
    return (Y, P) if return_p else Y


def naive_attention_rows_fp64(Q, K, V, scale=None, rows_per_chunk=1024):
    """FP64 naive attention (oracles.py:74-104 arithmetic) over query-row
    chunks, so every row of a long sequence can be checked without an n x n
    matrix in memory at once."""
    Q, K, V = (np.asarray(x, dtype=np.float64) for x in (Q, K, V))
    b, h, n_q, d = Q.shape
    sc = _scale(d) if scale is None else float(scale)
    Y = np.empty((b, h, n_q, V.shape[3]))
    for bi in range(b):
        for hi in range(h):
            for r0 in range(0, n_q, rows_per_chunk):
                s = (Q[bi, hi, r0:r0 + rows_per_chunk] @ K[bi, hi].T) * sc
                s -= s.max(axis=1, keepdims=True)
                np.exp(s, out=s)
                Y[bi, hi, r0:r0 + rows_per_chunk] = (s @ V[bi, hi]) / s.sum(axis=1, keepdims=True)
    return Y


def vectorized_probs(Q, K, scale=None, dtype=np.float32):
    """Probability matrix of the batched pipeline (oracles.py:107-122)."""
    dt = np.dtype(dtype)
    Q, K = (np.asarray(x).astype(dt, copy=False) for x in (Q, K))
    sc = dt.type(_scale(Q.shape[3]) if scale is None else scale)
    s = np.matmul(Q, K.transpose(0, 1, 3, 2)) * sc
    s -= s.max(axis=-1, keepdims=True)
    np.exp(s, out=s)
    s /= s.sum(axis=-1, keepdims=True)
    return s


def sampled_rows_fp64(Q, K, V, rows, scale=None):
    """FP64 outputs for selected rows ``rows = [(b, h, q), ...]``; returns an
    array (len(rows), d_v). Same arithmetic as naive_attention, one row at a
    time, so n may be far beyond what an n x n matrix allows."""
    d = Q.shape[3]
    sc = _scale(d) if scale is None else float(scale)
    out = np.empty((len(rows), V.shape[3]), dtype=np.float64)
    for r, (bi, hi, qi) in enumerate(rows):
        q = np.asarray(Q[bi, hi, qi], dtype=np.float64)
        Kh = np.asarray(K[bi, hi], dtype=np.float64)
        Vh = np.asarray(V[bi, hi], dtype=np.float64)
        s = (Kh @ q) * sc
        s -= s.max()
        np.exp(s, out=s)
        out[r] = (s @ Vh) / s.sum()
    return out


def partial_state_fp64(Q, K, V, kv_begin, kv_end, scale=None):
    """FP64 (m, S, W) of keys [kv_begin, kv_end) for every query row:
    m (b, h, n_q), S (b, h, n_q), W (b, h, n_q, d_v). An empty range is the
    identity (-inf, 0, 0)."""
    Q, K, V = (np.asarray(x, dtype=np.float64) for x in (Q, K, V))
    b, h, n_q, d = Q.shape
    d_v = V.shape[3]
    sc = _scale(d) if scale is None else float(scale)
    m = np.full((b, h, n_q), -np.inf)
    S = np.zeros((b, h, n_q))
    W = np.zeros((b, h, n_q, d_v))
    if kv_end <= kv_begin:
        return m, S, W
    for bi in range(b):
        for hi in range(h):
            s = (Q[bi, hi] @ K[bi, hi, kv_begin:kv_end].T) * sc
            mm = s.max(axis=1)
            p = np.exp(s - mm[:, None])
            m[bi, hi] = mm
            S[bi, hi] = p.sum(axis=1)
            W[bi, hi] = p @ V[bi, hi, kv_begin:kv_end]
    return m, S, W


def bound_threshold(n, block_size=128, slack=DEFAULT_SLACK):
    """u * L(n, B) * slack — verify.py:339-343."""
    return U32 * scan_depth(n, block_size) * slack


def row_err_conditioned(y, Q, K, V, ref=None, scale=None):
    """Per-row error scaled by the row's conditioning instead of |y|:
    ||y_hat - y||_2 / ||sum_j p_j |v_j| ||_2 with p the FP64 softmax row.
    Y is a convex combination of V rows, so this is the forward error of that
    combination relative to the magnitudes it combines; it stays meaningful
    when a narrow (d_v <= 2) output row cancels to ~0, where the relative
    error of row_rel_err is unbounded for any finite-precision method (the
    reference's own FP32 scan included). Test-only helper, FP64 throughout."""
    y = np.asarray(y, dtype=np.float64)
    if ref is None:
        ref = naive_attention(Q, K, V, scale=scale)
    _, P = naive_attention(Q, K, V, scale=scale, return_p=True)
    mag = np.matmul(P, np.abs(np.asarray(V, dtype=np.float64)))
    tiny = np.finfo(np.float64).tiny
    return np.linalg.norm(y - ref, axis=-1) / np.maximum(np.linalg.norm(mag, axis=-1), tiny)


def row_rel_err(y, ref):
    """Per-row relative L2 error against a reference (verify.py:336-338)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    tiny = np.finfo(np.float64).tiny
    return np.linalg.norm(y - ref, axis=-1) / np.maximum(np.linalg.norm(ref, axis=-1), tiny)
