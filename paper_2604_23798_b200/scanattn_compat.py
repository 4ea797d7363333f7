"""``scan_forward(problem, cfg)`` with the reference's signature, on the GPU.

Mirrors the public surface of the reference engine
(/root/reference/pkg/src/scanattn/__init__.py:6-65, engine.py:63-131,
engine.py:385-427) so the reference's own harnesses — ``verify.bound_check``
(verify.py:320-358, via its ``candidate=`` argument), ``drift_metrics``
(verify.py:142-215) and the CLI's verify flow — can consume outputs computed
by the sm_100a kernels:

* ``scan_forward(problem, cfg) -> (AttentionOutput, ScanTrace | None)``
  accepts a reference ``AttentionProblem`` (duck-typed: ``.Q/.K/.V`` with a
  numpy ``.data`` array, ``.scale``) or this module's ``AttentionProblem``.
* ``cfg.precision`` must be FP32: the GPU path has no FP64 kernel and no CPU
  fallback, so FP64 raises :class:`ShapeError` (engine.py:392-393 raises the
  same type for an invalid config).
* ``cfg.block_size`` is the reference's B; it sets the depth bound
  L(n, B) reported in the trace (engine.py:47-55). ``cfg.workers`` is
  accepted and ignored (the reference's output is worker-invariant too,
  engine.py:11-13). ``cfg.tile_q`` is accepted; the kernel's query tile is
  fixed by its launch configuration.
* The returned ``Y`` is a ``Tensor4`` of the problem's own class when the
  problem came from the reference (so reference type checks pass), else of
  this module's minimal ``Tensor4``.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import attention as _att
from .attention import attention_from_host, resolve_kv_splits, scaled_dot_product_attention
from .errors import ShapeError

__all__ = [
    "Precision",
    "Tensor4",
    "AttentionProblem",
    "AttentionOutput",
    "ScanConfig",
    "ScanTrace",
    "scan_depth",
    "depth_cap",
    "scan_forward",
    "analytic_trace",
    "StateTriple",
    "blockwise_states",
    "inter_block_combine",
    "block_validation",
    "BlockValidationReport",
]


class Precision(enum.Enum):
    """Same values as monoid.Precision (monoid.py:38-70)."""

    FP32 = "fp32"
    FP64 = "fp64"

    @property
    def dtype(self):
        return np.dtype(np.float32) if self is Precision.FP32 else np.dtype(np.float64)

    @property
    def unit_roundoff(self):
        return 2.0 ** -24 if self is Precision.FP32 else 2.0 ** -53


class Tensor4:
    """(b, h, n, width) contiguous finite array (tensorio.py:46-80)."""

    def __init__(self, data, precision=None):
        data = np.asarray(data)
        if data.ndim != 4:
            raise ShapeError(f"expected 4 axes (b, h, n, width), got shape {data.shape}")
        if precision is None:
            precision = Precision.FP32 if data.dtype == np.float32 else Precision.FP64
        data = np.ascontiguousarray(data, dtype=np.dtype(precision.value.replace("fp", "float")))
        if not np.all(np.isfinite(data)):
            raise ShapeError("tensor elements must all be finite")
        self.data = data
        self.precision = precision

    @property
    def dims(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype


@dataclass
class AttentionProblem:
    """Q, K, V and the derived 1/sqrt(d) scale (tensorio.py:83-112)."""

    Q: Tensor4
    K: Tensor4
    V: Tensor4

    def __post_init__(self):
        b, h, n, d = self.Q.dims
        if self.K.dims != (b, h, n, d):
            raise ShapeError(f"K dims {self.K.dims} != Q dims {self.Q.dims}")
        if self.V.dims[:3] != (b, h, n):
            raise ShapeError(f"V dims {self.V.dims[:3]} disagree with Q on (b, h, n)")

    @property
    def dims(self):
        b, h, n, d = self.Q.dims
        return b, h, n, d, self.V.dims[3]

    @property
    def precision(self):
        return self.Q.precision

    @property
    def scale(self):
        return 1.0 / float(np.sqrt(self.Q.dims[3]))


@dataclass
class AttentionOutput:
    """Y always; P is never produced by the scan path (oracles.py:36-45)."""

    Y: object
    P: object = None

    @property
    def precision(self):
        return self.Y.precision


@dataclass(frozen=True)
class ScanConfig:
    """engine.py:63-89, with the precision defaulting to FP32 (the only
    precision the GPU path computes in) and ``kv_splits`` added (0 = auto)."""

    block_size: int = 128
    tile_q: int = 64
    workers: int | str = 1
    precision: object = Precision.FP32
    trace: bool = False
    kv_splits: int = 0

    def __post_init__(self):
        for name in ("block_size", "tile_q"):
            if getattr(self, name) < 1:
                raise ShapeError(f"ScanConfig.{name} = {getattr(self, name)}: needs a "
                                 "positive tile size")
        w = self.workers
        if not (w == "auto" or (isinstance(w, int) and w >= 1)):
            raise ShapeError(f"ScanConfig.workers = {w!r}: use 'auto' or a count >= 1 "
                             "(ignored on the GPU)")
        if self.kv_splits < 0:
            raise ShapeError(f"ScanConfig.kv_splits = {self.kv_splits}: use 0 (auto) or a "
                             "split count")


@dataclass
class ScanTrace:
    """Analytic trace of the GPU schedule (fields as engine.py:92-131).

    ``leaf_count`` counts score evaluations (one per query-key pair);
    ``merge_count`` counts (m,S,W) state combines: one per key tile folded into
    a running row state plus the split-tree merges; ``critical_depth`` is the
    reference's bound L(n, B) for ``cfg.block_size`` (the figure the FP32 error
    threshold is built from, engine.py:47-55); ``schedule_depth`` is this
    schedule's own combine depth: the 16-lane max butterfly (4) + the longest
    tile chain + ceil(log2 splits). ``peak_extra_memory`` is the split
    workspace in bytes.
    """

    merge_count: int = 0
    critical_depth: int = 0
    per_level_counts: list = field(default_factory=list)
    leaf_count: int = 0
    peak_extra_memory: int = 0
    n_paths: int = 0
    schedule_depth: int = 0
    kv_splits: int = 1

    @property
    def merges_per_query(self):
        return self.merge_count / self.n_paths if self.n_paths else 0.0


def _clog2(x):
    return 0 if x <= 1 else int(math.ceil(math.log2(x)))


def scan_depth(n, block_size):
    """engine.py:47-55."""
    if n < 1 or block_size < 1:
        raise ShapeError("n and block_size must be >= 1")
    return _clog2(min(block_size, n)) + 2 * _clog2(-(-n // block_size)) + 3


def depth_cap(n):
    """engine.py:58-60."""
    return 2 * _clog2(n) + 3


KEY_TILE = 64  # keys per tile in the forward kernel (FwdTraits::TK; 32 for d > 128)


def _precision_name(p):
    return getattr(p, "value", str(p)).lower()


def analytic_trace(b, h, n, block_size, splits, workspace_bytes=None, d_v=64,
                   key_tile=KEY_TILE):
    """ScanTrace of the GPU schedule for a (b, h, n) problem run with
    ``splits`` KV splits and ``key_tile`` keys per tile (see
    :class:`ScanTrace`); ``workspace_bytes`` is the split workspace the
    library asked for (elsa_workspace_bytes), else the unbatched size."""
    tiles = -(-n // key_tile)
    tps = -(-tiles // splits)
    paths = b * h * n
    return ScanTrace(
        merge_count=paths * (tiles + splits - 1),
        critical_depth=scan_depth(n, block_size),
        per_level_counts=[paths * tiles] + ([paths * (splits - 1)] if splits > 1 else []),
        leaf_count=b * h * n * n,
        peak_extra_memory=(int(workspace_bytes) if workspace_bytes is not None
                           else (splits * b * h * n * (2 + 64 * -(-d_v // 64)) * 4) if splits > 1 else 0),
        n_paths=paths,
        schedule_depth=4 + tps + _clog2(splits),
        kv_splits=splits,
    )


def scan_forward(problem, cfg=None, device=None):
    """GPU ``scan_forward``: returns ``(AttentionOutput, ScanTrace | None)``."""
    cfg = ScanConfig() if cfg is None else cfg
    if not hasattr(cfg, "precision") or not hasattr(cfg, "block_size"):
        raise ShapeError("cfg must be a ScanConfig")
    if _precision_name(cfg.precision) != "fp32":
        raise ShapeError("the GPU scan path computes in FP32 only; FP64 has no kernel and "
                         "there is no CPU fallback")
    Qd, Kd, Vd = problem.Q.data, problem.K.data, problem.V.data
    b, h, n, d = Qd.shape
    d_v = Vd.shape[3]
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    splits_req = int(getattr(cfg, "kv_splits", 0))
    # host arrays in, host Y out: the pipelined host entry point (copies overlap the kernels)
    q, k, v = (torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)) for x in (Qd, Kd, Vd))
    Y = attention_from_host(q, k, v, scale=float(problem.scale), kv_splits=splits_req, device=dev,
                            check_numerics=True).numpy()
    t4_cls = type(problem.Q)
    prec = problem.Q.precision if hasattr(problem.Q, "precision") else Precision.FP32
    try:
        y_t4 = t4_cls(Y, prec) if _precision_name(prec) == "fp32" else Tensor4(Y, Precision.FP32)
    except Exception:  # a foreign Tensor4 with another constructor
        y_t4 = Tensor4(Y, Precision.FP32)
    out = AttentionOutput(y_t4)
    trace = None
    if getattr(cfg, "trace", False):
        plan = _att.describe_plan(q, k, v, splits_req)  # "<cfg> tq=.. tk=.. kv_splits=.."
        tk = int(plan.split("tk=")[1].split()[0])
        trace = analytic_trace(b, h, n, cfg.block_size, resolve_kv_splits(q, k, v, splits_req),
                               _att.workspace_bytes(q, k, v, splits_req), d_v=d_v, key_tile=tk)
    return out, trace


# ---------------------------------------------------------------------------
# Block-level surface: engine.blockwise_states,
# engine.inter_block_combine and verify.block_validation on device states.


@dataclass(frozen=True)
class StateTriple:
    """(m, S, W) summary of one key range (monoid.py:73-120), host copy."""

    m: float
    S: float
    W: np.ndarray

    def is_identity(self):
        return bool(np.isneginf(self.m))


def _triples(m, S, W):
    return [StateTriple(np.float32(a), np.float32(b), np.asarray(c, dtype=np.float32))
            for a, b, c in zip(m, S, W)]


def _problem_tensors(problem, dev):
    return tuple(torch.from_numpy(np.ascontiguousarray(t.data, dtype=np.float32)).to(dev)
                 for t in (problem.Q, problem.K, problem.V))


def blockwise_states(problem, cfg, query_index, b_idx=0, h_idx=0, block_size=None, device=None):
    """Per-block totals for one query (engine.py:430-451), computed by the
    sm_100a blockwise kernel (elsa_blockwise_f32). ``block_size`` overrides
    ``cfg.block_size``; returns a list of :class:`StateTriple`."""
    B = cfg.block_size if block_size is None else int(block_size)
    if B < 1:
        raise ShapeError(f"block size must be >= 1, got {B}")
    b, h, n, d = problem.Q.data.shape
    if not (0 <= query_index < n):
        raise ShapeError(f"query index {query_index} out of range [0, {n})")
    if _precision_name(getattr(cfg, "precision", Precision.FP32)) != "fp32":
        raise ShapeError("the GPU block path computes in FP32 only")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    q, k, v = _problem_tensors(problem, dev)
    qi = q[b_idx:b_idx + 1, h_idx:h_idx + 1, query_index:query_index + 1]
    m, S, W = _att.blockwise_states(qi, k[b_idx:b_idx + 1, h_idx:h_idx + 1],
                                    v[b_idx:b_idx + 1, h_idx:h_idx + 1], block_size=B,
                                    scale=float(problem.scale))
    return _triples(m[0, 0, 0].cpu().numpy(), S[0, 0, 0].cpu().numpy(), W[0, 0, 0].cpu().numpy())


def inter_block_combine(block_totals, return_prefixes=False, device=None):
    """engine.py:265-297 on the device: the up-sweep total and, optionally,
    the exclusive prefixes (identity first)."""
    totals = list(block_totals)
    if not totals:
        raise ShapeError("no block totals to combine")
    widths = {np.asarray(t.W).shape[0] for t in totals}
    if len(widths) != 1:
        raise ShapeError(f"mixed value widths {sorted(widths)}")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    m = torch.tensor([[float(t.m) for t in totals]], dtype=torch.float32, device=dev)
    S = torch.tensor([[float(t.S) for t in totals]], dtype=torch.float32, device=dev)
    W = torch.from_numpy(np.stack([np.asarray(t.W, dtype=np.float32) for t in totals])[None]).to(dev)
    res = _att.inter_block_combine(m, S, W, return_prefixes=return_prefixes)
    (tm, tS, tW), pre = (res if return_prefixes else (res, None))
    total = StateTriple(np.float32(tm[0].item()), np.float32(tS[0].item()), tW[0].cpu().numpy())
    if not return_prefixes:
        return total
    return total, _triples(pre[0][0].cpu().numpy(), pre[1][0].cpu().numpy(), pre[2][0].cpu().numpy())


_TINY = np.finfo(np.float64).tiny


def _state_signature(t):
    """(m, S, W..., W/S...) of a state as one float64 vector."""
    w = np.asarray(t.W, dtype=np.float64).ravel()
    s = float(t.S)
    return np.hstack((float(t.m), s, w, w / max(s, _TINY)))


def _triple_rel_dev(t1, t2):
    """Largest componentwise relative difference of two states over
    (m, S, W, W/S) — the deviation verify.py:218-227 defines."""
    a, b = _state_signature(t1), _state_signature(t2)
    return float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), _TINY)).max())


class BlockValidationReport:
    """Result of :func:`block_validation`; same attributes, ``passed`` and
    ``to_dict`` as the reference's report (verify.py:230-246)."""

    _FIELDS = ("partitions", "query_points", "max_pairwise_dev", "max_vs_sequential_dev",
               "per_partition_dev")

    def __init__(self, partitions, query_points, max_pairwise_dev, max_vs_sequential_dev,
                 per_partition_dev):
        self.partitions = partitions
        self.query_points = query_points
        self.max_pairwise_dev = max_pairwise_dev
        self.max_vs_sequential_dev = max_vs_sequential_dev
        self.per_partition_dev = per_partition_dev

    def passed(self, tol):
        return max(self.max_pairwise_dev, self.max_vs_sequential_dev) <= tol

    def to_dict(self):
        conv = {"partitions": list,
                "query_points": lambda pts: [list(p) for p in pts],
                "per_partition_dev": lambda dv: {str(k): x for k, x in dv.items()}}
        return {f: conv.get(f, lambda x: x)(getattr(self, f)) for f in self._FIELDS}


def block_validation(problem, cfg, partitions, query_indices=None, device=None):
    """verify.block_validation (verify.py:249-282) on device states: for each
    partition size the per-block states of every query come from
    elsa_blockwise_f32 and their totals from the device up-sweep
    (elsa_block_scan_f32); totals are compared pairwise and against the
    whole-range single-chain state (elsa_partial_f32 with one split, the GPU
    path's own left-to-right fold, standing in for the reference's per-key
    sequential fold)."""
    partitions = [int(p) for p in partitions]
    if any(p < 1 for p in partitions):
        raise ShapeError("partition block sizes must be >= 1")
    b, h, n, d = problem.Q.data.shape
    if query_indices is None:
        query_indices = sorted({0, n // 3, (2 * n) // 3, n - 1})
    heads = sorted({(0, 0), (b - 1, h - 1)})
    points = [(bi, hi, qi) for (bi, hi) in heads for qi in query_indices]
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    q, k, v = _problem_tensors(problem, dev)
    sc = float(problem.scale)
    seq_m, seq_S, seq_W = _att.partial_states(q, k, v, scale=sc, kv_splits=1)
    totals_by_p = {}
    for p in partitions:
        m, S, W = _att.blockwise_states(q, k, v, block_size=p, scale=sc)
        totals_by_p[p] = tuple(t.cpu().numpy() for t in _att.inter_block_combine(m, S, W))
    max_pair = max_seq = 0.0
    per_partition = {p: 0.0 for p in partitions}
    for bi, hi, qi in points:
        seq = StateTriple(seq_m[bi, hi, qi].item(), seq_S[bi, hi, qi].item(),
                          seq_W[bi, hi, qi].cpu().numpy())
        tot = [StateTriple(*(a[bi, hi, qi] for a in totals_by_p[p])) for p in partitions]
        for i, t1 in enumerate(tot):
            dev_ = _triple_rel_dev(t1, seq)
            max_seq = max(max_seq, dev_)
            per_partition[partitions[i]] = max(per_partition[partitions[i]], dev_)
            for t2 in tot[i + 1:]:
                max_pair = max(max_pair, _triple_rel_dev(t1, t2))
    return BlockValidationReport(partitions, points, max_pair, max_seq, per_partition)
