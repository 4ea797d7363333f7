"""(m, S, W) monoid restated in numpy — oracle only.

Follows /root/reference/pkg/src/scanattn/monoid.py:
  * combine arithmetic and identity guard: merge_lanes_into, monoid.py:160-200
    (m = max; f_x = exp(m_x - m) with the both-identity NaN forced to
    exp(-inf) = 0; W = W_a f_a + W_b f_b; S = S_a f_a + S_b f_b, products
    rounded before the add — separate numpy ufuncs, no FMA);
  * scalar merge with identity short-circuit: merge, monoid.py:214-231;
  * balanced pairwise tree, odd tail passes through: merge_tree,
    monoid.py:234-265.
States are plain tuples ``(m, S, W)`` of numpy scalars/arrays in one dtype.
"""

from __future__ import annotations

import numpy as np

__all__ = ["identity_state", "merge_lanes", "merge", "merge_tree"]


def identity_state(d_v, dtype=np.float64):
    """(-inf, 0, 0) — monoid.py:122-125."""
    dt = np.dtype(dtype)
    return dt.type(-np.inf), dt.type(0.0), np.zeros(d_v, dtype=dt)


def merge_lanes(m_a, S_a, W_a, m_b, S_b, W_b):
    """Lane-wise guarded combine (monoid.py:160-200). ``m_*, S_*`` share a
    shape X, ``W_*`` is X + (d_v,). Returns new arrays."""
    m_a, m_b = np.asarray(m_a), np.asarray(m_b)
    m = np.maximum(m_a, m_b)
    with np.errstate(invalid="ignore"):
        da = np.subtract(m_a, m)
        db = np.subtract(m_b, m)
    # (-inf) - (-inf) = NaN only when both sides are the identity
    da = np.where(np.isnan(da), -np.inf, da).astype(m.dtype, copy=False)
    db = np.where(np.isnan(db), -np.inf, db).astype(m.dtype, copy=False)
    fa = np.exp(da)
    fb = np.exp(db)
    W = np.multiply(W_a, fa[..., None])
    W = np.add(W, np.multiply(W_b, fb[..., None]))
    S = np.add(np.multiply(S_a, fa), np.multiply(S_b, fb))
    return m, S, W


def merge(a, b):
    """Scalar combine with the identity short-circuit (monoid.py:214-231)."""
    ma, Sa, Wa = a
    mb, Sb, Wb = b
    if np.isneginf(ma):
        return b
    if np.isneginf(mb):
        return a
    m, S, W = merge_lanes(np.asarray(ma)[None], np.asarray(Sa)[None], np.asarray(Wa)[None],
                          np.asarray(mb)[None], np.asarray(Sb)[None], np.asarray(Wb)[None])
    return m[0], S[0], W[0]


def merge_tree(states, d_v=None, dtype=np.float64):
    """Balanced pairwise reduction, odd tail passes through (monoid.py:234-265).
    ``states`` is a sequence of (m, S, W); the empty sequence gives the
    identity."""
    states = list(states)
    if not states:
        return identity_state(0 if d_v is None else d_v, dtype)
    if len(states) == 1:
        return states[0]
    dt = np.asarray(states[0][2]).dtype
    m = np.array([s[0] for s in states], dtype=dt)
    S = np.array([s[1] for s in states], dtype=dt)
    W = np.stack([np.asarray(s[2], dtype=dt) for s in states])
    while m.shape[0] > 1:
        k = m.shape[0]
        pairs = k // 2
        nm, nS, nW = merge_lanes(m[0:2 * pairs:2], S[0:2 * pairs:2], W[0:2 * pairs:2],
                                 m[1:2 * pairs:2], S[1:2 * pairs:2], W[1:2 * pairs:2])
        if k % 2:
            nm = np.concatenate([nm, m[-1:]])
            nS = np.concatenate([nS, S[-1:]])
            nW = np.concatenate([nW, W[-1:]])
        m, S, W = nm, nS, nW
    return m[0], S[0], W[0]
