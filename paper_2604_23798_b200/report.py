"""``scanattn-bench-v1`` records and the scaling fit for GPU runs
(SURVEY §8f row 4).

Mirrors /root/reference/pkg/src/scanattn/bench.py so GPU measurements land in
the same report schema the reference's CLI writes (``scanattn bench
--report``, cli.py:231-265):

* :class:`BenchRecord` — same fields, JSON/CSV serialisation and derived
  median/p5/p95 (bench.py:40-110);
* :func:`fit_scaling` — least squares of latency on [L(n, B), n^2, 1] with
  normalised columns and the relative RMS residual (bench.py:193-219);
* :func:`emit_report` — the JSON document + flat CSV (bench.py:222-242);
* :func:`nearest_rank_percentiles` — verify.py:54-66;
* :func:`run_bench` — one workload timed on the device: every repeat is one
  ``scaled_dot_product_attention`` call bracketed by CUDA events on the
  launching stream (the reference times host wall clock, bench.py:175-181).
  Modes: ``scan`` (this library's FP32 kernels, merge/leaf counts attached
  from the analytic trace), ``scan16`` (the bf16 tcgen05 kernel) and
  ``sdpa`` (torch's own SDPA on the same inputs, a GPU comparator in place of
  the reference's CPU ``naive``/``seq`` modes).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ShapeError

__all__ = [
    "BenchRecord",
    "ScalingFit",
    "nearest_rank_percentiles",
    "fit_scaling",
    "emit_report",
    "run_bench",
    "MODES",
]

MODES = ("scan", "scan16", "sdpa")


def nearest_rank_percentiles(samples):
    """Median / p95 / p99 by the nearest-rank rule (verify.py:54-66)."""
    s = np.sort(np.asarray(samples, dtype=np.float64).ravel())
    if s.size == 0:
        return {"median": 0.0, "p95": 0.0, "p99": 0.0}

    def rank(p):
        return s[max(math.ceil(p / 100.0 * s.size), 1) - 1]

    return {"median": float(rank(50)), "p95": float(rank(95)), "p99": float(rank(99))}


def _clog2(x):
    return 0 if x <= 1 else int(math.ceil(math.log2(x)))


def _scan_depth(n, block_size):
    return _clog2(min(block_size, n)) + 2 * _clog2(-(-n // block_size)) + 3


@dataclass
class BenchRecord:
    """One benchmarked workload (bench.py:40-110); latencies in seconds."""

    mode: str
    n: int
    block_size: int
    tile_q: int
    d: int
    d_v: int
    b: int
    h: int
    precision: str
    repeats: int
    warmup: int
    latencies: list = field(default_factory=list)
    merge_count: int = 0
    leaf_count: int = 0
    peak_extra_memory: int = 0
    status: str = "ok"
    error: str = ""

    def summary(self):
        if not self.latencies:
            return {"median": None, "p5": None, "p95": None}
        s = np.sort(np.asarray(self.latencies))
        pct = nearest_rank_percentiles(s)
        idx5 = max(int(np.ceil(0.05 * s.size)), 1) - 1
        return {"median": float(pct["median"]), "p5": float(s[idx5]), "p95": float(pct["p95"])}

    def to_dict(self):
        out = {
            "mode": self.mode, "n": self.n, "block_size": self.block_size,
            "tile_q": self.tile_q, "d": self.d, "d_v": self.d_v,
            "b": self.b, "h": self.h, "precision": self.precision,
            "repeats": self.repeats, "warmup": self.warmup,
            "latencies": [float(x) for x in self.latencies],
            "merge_count": self.merge_count, "leaf_count": self.leaf_count,
            "peak_extra_memory": self.peak_extra_memory,
            "status": self.status, "error": self.error,
        }
        out.update({f"latency_{k}": v for k, v in self.summary().items()})
        return out

    CSV_FIELDS = (
        "mode", "n", "block_size", "tile_q", "d", "d_v", "b", "h", "precision",
        "repeats", "warmup", "status", "latency_median", "latency_p5", "latency_p95",
        "merge_count", "leaf_count", "peak_extra_memory",
    )

    @classmethod
    def csv_header(cls):
        return ",".join(cls.CSV_FIELDS)

    def csv_row(self):
        d = self.to_dict()
        return ",".join("" if d[f] is None else (repr(d[f]) if isinstance(d[f], float) else str(d[f]))
                        for f in self.CSV_FIELDS)


@dataclass
class ScalingFit:
    """a * L(n, B) + b * n^2 + c with its relative RMS residual (bench.py:113-130)."""

    a: float
    b: float
    c: float
    residual: float
    block_size: int
    points: list

    def predict(self, n):
        return self.a * _scan_depth(int(n), self.block_size) + self.b * float(n) ** 2 + self.c

    def to_dict(self):
        return {
            "a": self.a, "b": self.b, "c": self.c,
            "residual": self.residual, "block_size": self.block_size,
            "points": [[int(n), float(t)] for n, t in self.points],
        }


def fit_scaling(points, block_size):
    """Ordinary least squares of latency on [L(n, B), n^2, 1], columns
    normalised before the solve (bench.py:193-219)."""
    pts = [(int(n), float(t)) for n, t in points]
    ns = np.array([p[0] for p in pts], dtype=np.float64)
    ts = np.array([p[1] for p in pts], dtype=np.float64)
    if len(set(ns.tolist())) < 3:
        raise ShapeError("need at least 3 points with distinct n to fit 3 coefficients")
    design = np.stack([
        np.array([_scan_depth(int(n), block_size) for n in ns], dtype=np.float64),
        ns ** 2,
        np.ones_like(ns),
    ], axis=1)
    norms = np.linalg.norm(design, axis=0)
    coef, *_ = np.linalg.lstsq(design / norms, ts, rcond=None)
    coef = coef / norms
    pred = design @ coef
    denom = max(float(np.linalg.norm(ts)), np.finfo(np.float64).tiny)
    return ScalingFit(a=float(coef[0]), b=float(coef[1]), c=float(coef[2]),
                      residual=float(np.linalg.norm(pred - ts) / denom),
                      block_size=block_size, points=pts)


def emit_report(records, fits, json_path, csv_path=None):
    """JSON report + flat CSV (bench.py:222-242)."""
    doc = {
        "schema": "scanattn-bench-v1",
        "records": [r.to_dict() for r in records],
        "fits": [f.to_dict() for f in fits],
    }
    with open(json_path, "w") as f:
        json.dump(doc, f, indent=2)
        f.write("\n")
    if csv_path is None:
        csv_path = str(json_path).rsplit(".", 1)[0] + ".csv"
    with open(csv_path, "w") as f:
        f.write(BenchRecord.csv_header() + "\n")
        for r in records:
            f.write(r.csv_row() + "\n")
    return json_path, csv_path


def run_bench(b, h, n, d=64, d_v=64, mode="scan", repeats=20, warmup=3, block_size=128,
              seed=0, device=None, flush_l2=True):
    """Time one workload on the device; returns a :class:`BenchRecord`.

    Inputs are N(0, 1) draws made on the device (seeded). Each repeat is one
    call bracketed by CUDA events on the current stream; with ``flush_l2`` a
    256 MiB buffer is rewritten before every repeat so no repeat reads the
    previous one's operands from L2.
    """
    import torch

    from . import attention as att
    from .scanattn_compat import analytic_trace

    if mode not in MODES:
        raise ShapeError(f"unknown bench mode {mode!r}; use one of {MODES}")
    if repeats < 3:
        raise ShapeError(f"repeats must be >= 3, got {repeats}")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    dt = torch.bfloat16 if mode == "scan16" else torch.float32
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    q = torch.randn(b, h, n, d, device=dev, generator=g).to(dt)
    k = torch.randn(b, h, n, d, device=dev, generator=g).to(dt)
    v = torch.randn(b, h, n, d_v, device=dev, generator=g).to(dt)
    rec = BenchRecord(mode=mode, n=n, block_size=block_size, tile_q=64, d=d, d_v=d_v, b=b, h=h,
                      precision="bf16" if mode == "scan16" else "fp32", repeats=repeats,
                      warmup=warmup)
    if mode == "sdpa":
        fn = (lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
    else:
        fn = (lambda: att.scaled_dot_product_attention(q, k, v))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_l2 else None
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    for _ in range(repeats):
        if flush is not None:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        rec.latencies.append(e0.elapsed_time(e1) * 1e-3)
    if mode == "scan":
        splits = att.resolve_kv_splits(q, k, v, 0)
        tr = analytic_trace(b, h, n, block_size, splits, att.workspace_bytes(q, k, v, 0))
        rec.merge_count, rec.leaf_count = tr.merge_count, tr.leaf_count
        rec.peak_extra_memory = tr.peak_extra_memory
    return rec
