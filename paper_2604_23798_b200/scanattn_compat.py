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

from .attention import resolve_kv_splits, scaled_dot_product_attention
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
        if self.block_size < 1:
            raise ShapeError(f"block_size must be >= 1, got {self.block_size}")
        if self.tile_q < 1:
            raise ShapeError(f"tile_q must be >= 1, got {self.tile_q}")
        if self.workers != "auto" and (not isinstance(self.workers, int) or self.workers < 1):
            raise ShapeError(f"workers must be a positive integer or 'auto', got {self.workers!r}")
        if self.kv_splits < 0:
            raise ShapeError("kv_splits must be >= 0")


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


KEY_TILE = 64  # keys per tile in the forward kernel (FwdTraits::TK)


def _precision_name(p):
    return getattr(p, "value", str(p)).lower()


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
    q = torch.from_numpy(np.ascontiguousarray(Qd, dtype=np.float32)).to(dev)
    k = torch.from_numpy(np.ascontiguousarray(Kd, dtype=np.float32)).to(dev)
    v = torch.from_numpy(np.ascontiguousarray(Vd, dtype=np.float32)).to(dev)
    splits_req = int(getattr(cfg, "kv_splits", 0))
    y = scaled_dot_product_attention(q, k, v, scale=float(problem.scale), kv_splits=splits_req,
                                     check_numerics=True)
    Y = y.cpu().numpy()
    t4_cls = type(problem.Q)
    prec = problem.Q.precision if hasattr(problem.Q, "precision") else Precision.FP32
    try:
        y_t4 = t4_cls(Y, prec) if _precision_name(prec) == "fp32" else Tensor4(Y, Precision.FP32)
    except Exception:  # a foreign Tensor4 with another constructor
        y_t4 = Tensor4(Y, Precision.FP32)
    out = AttentionOutput(y_t4)
    trace = None
    if getattr(cfg, "trace", False):
        splits = resolve_kv_splits(q, k, v, splits_req)
        tiles = -(-n // KEY_TILE)
        tps = -(-tiles // splits)
        paths = b * h * n
        trace = ScanTrace(
            merge_count=paths * (tiles + splits - 1),
            critical_depth=scan_depth(n, cfg.block_size),
            per_level_counts=[paths * tiles] + ([paths * (splits - 1)] if splits > 1 else []),
            leaf_count=b * h * n * n,
            peak_extra_memory=(splits * b * h * n * (2 + 64) * 4) if splits > 1 else 0,
            n_paths=paths,
            schedule_depth=4 + tps + _clog2(splits),
            kv_splits=splits,
        )
    return out, trace
