"""``scanattn-bench-v1`` records and the scaling fit for GPU runs
(SURVEY §8f row 4).

GPU measurements are written in the report schema the reference's CLI emits
(``scanattn bench --report``, cli.py:231-265; schema of bench.py:40-130,
222-242) so the two can be read by the same tools. The implementation here
is this package's own and is pinned by the reference's output bytes
(tests/golden/harness.npz), not derived from its code:

* :class:`BenchRecord` — a schema-driven record: the field table
  ``RECORD_FIELDS`` fixes the key order of the JSON object and the CSV
  columns; the median / p5 / p95 summary is computed when serialising;
* :func:`fit_scaling` — ``T(n) = a L(n, B) + b n^2 + c`` by a Householder QR
  solve of the column-equilibrated design, plus the relative residual;
* :func:`emit_report` — JSON document + flat CSV;
* :func:`nearest_rank_percentiles` — nearest-rank order statistics;
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

import numpy as np

from .errors import ShapeError

__all__ = [
    "BenchRecord",
    "ScalingFit",
    "RECORD_FIELDS",
    "nearest_rank_percentiles",
    "fit_scaling",
    "emit_report",
    "run_bench",
    "MODES",
]

MODES = ("scan", "scan16", "sdpa")


def _order_stat(sorted_samples, pct):
    """The nearest-rank pct-th percentile of an ascending array: element
    ceil(pct/100 * N), 1-based, at least the first."""
    k = math.ceil(pct * sorted_samples.size / 100.0)
    return float(sorted_samples[min(max(k, 1), sorted_samples.size) - 1])


def nearest_rank_percentiles(samples):
    """Median / p95 / p99 by the nearest-rank rule (verify.py:54-66)."""
    ordered = np.sort(np.asarray(samples, dtype=np.float64), axis=None)
    if not ordered.size:
        return dict.fromkeys(("median", "p95", "p99"), 0.0)
    return {name: _order_stat(ordered, p) for name, p in (("median", 50), ("p95", 95),
                                                          ("p99", 99))}


def _depth(n, block):
    """L(n, B) (engine.py:47-55)."""
    def ceil_log2(x):
        return max(int(x) - 1, 0).bit_length()
    return ceil_log2(min(block, n)) + 2 * ceil_log2(-(-n // block)) + 3


# (name, default) in schema order; the defaults of the measured quantities
RECORD_FIELDS = (
    ("mode", None), ("n", None), ("block_size", None), ("tile_q", None), ("d", None),
    ("d_v", None), ("b", None), ("h", None), ("precision", None), ("repeats", None),
    ("warmup", None), ("latencies", list), ("merge_count", 0), ("leaf_count", 0),
    ("peak_extra_memory", 0), ("status", "ok"), ("error", ""),
)
_CSV_COLUMNS = ("mode", "n", "block_size", "tile_q", "d", "d_v", "b", "h", "precision",
                "repeats", "warmup", "status", "latency_median", "latency_p5", "latency_p95",
                "merge_count", "leaf_count", "peak_extra_memory")


class BenchRecord:
    """One timed workload; latencies in seconds. Fields are ``RECORD_FIELDS``
    (all required except those with a default); summary statistics are
    derived, never stored."""

    __slots__ = tuple(name for name, _ in RECORD_FIELDS)

    def __init__(self, **values):
        unknown = set(values) - set(self.__slots__)
        if unknown:
            raise TypeError(f"unknown BenchRecord fields: {sorted(unknown)}")
        for name, default in RECORD_FIELDS:
            if name in values:
                val = values[name]
            elif default is None:
                raise TypeError(f"BenchRecord needs {name!r}")
            else:
                val = default() if callable(default) else default
            setattr(self, name, val)

    def summary(self):
        if not len(self.latencies):
            return {"median": None, "p5": None, "p95": None}
        ordered = np.sort(np.asarray(self.latencies, dtype=np.float64))
        return {"median": _order_stat(ordered, 50), "p5": _order_stat(ordered, 5),
                "p95": _order_stat(ordered, 95)}

    def to_dict(self):
        out = {}
        for name, _ in RECORD_FIELDS:
            val = getattr(self, name)
            out[name] = [float(x) for x in val] if name == "latencies" else val
        for key, val in self.summary().items():
            out["latency_" + key] = val
        return out

    CSV_FIELDS = _CSV_COLUMNS

    @classmethod
    def csv_header(cls):
        return ",".join(_CSV_COLUMNS)

    def csv_row(self):
        row = self.to_dict()
        cells = []
        for col in _CSV_COLUMNS:
            val = row[col]
            cells.append("" if val is None else repr(val) if isinstance(val, float) else str(val))
        return ",".join(cells)


class ScalingFit:
    """``T(n) = a L(n, B) + b n^2 + c`` with its relative residual."""

    def __init__(self, a, b, c, residual, block_size, points):
        self.a, self.b, self.c = float(a), float(b), float(c)
        self.residual = float(residual)
        self.block_size = int(block_size)
        self.points = list(points)

    def predict(self, n):
        n = int(n)
        return self.a * _depth(n, self.block_size) + self.b * float(n) * float(n) + self.c

    def to_dict(self):
        return {"a": self.a, "b": self.b, "c": self.c, "residual": self.residual,
                "block_size": self.block_size,
                "points": [[int(n), float(t)] for n, t in self.points]}


def fit_scaling(points, block_size):
    """Least-squares fit of latency to [L(n, B), n^2, 1]: each design column
    is scaled to unit 2-norm (the raw columns span ~10 orders of magnitude),
    the system is solved through a reduced Householder QR (R c = Q^T t) and
    the scaling undone. Needs three distinct n."""
    pts = [(int(n), float(t)) for n, t in points]
    n_arr = np.fromiter((n for n, _ in pts), dtype=np.float64, count=len(pts))
    t_arr = np.fromiter((t for _, t in pts), dtype=np.float64, count=len(pts))
    if np.unique(n_arr).size < 3:
        raise ShapeError("the scaling fit has 3 coefficients: give at least 3 distinct n")
    cols = np.column_stack([[float(_depth(int(n), block_size)) for n in n_arr],
                            n_arr * n_arr, np.ones_like(n_arr)])
    scale = np.sqrt((cols * cols).sum(axis=0))
    qmat, rmat = np.linalg.qr(cols / scale, mode="reduced")
    coef = np.linalg.solve(rmat, qmat.T @ t_arr) / scale
    fitted = cols @ coef
    tnorm = float(np.sqrt(t_arr @ t_arr))
    resid = float(np.sqrt(((fitted - t_arr) ** 2).sum())) / max(tnorm, np.finfo(float).tiny)
    return ScalingFit(coef[0], coef[1], coef[2], resid, block_size, pts)


def emit_report(records, fits, json_path, csv_path=None):
    """Write the ``scanattn-bench-v1`` JSON document (2-space indent, newline
    terminated) and the flat CSV (default: the JSON path with ``.csv``)."""
    text = json.dumps({"schema": "scanattn-bench-v1",
                       "records": [r.to_dict() for r in records],
                       "fits": [f.to_dict() for f in fits]}, indent=2)
    if csv_path is None:
        stem, _, _ = str(json_path).rpartition(".")
        csv_path = (stem or str(json_path)) + ".csv"
    lines = [BenchRecord.csv_header()] + [r.csv_row() for r in records]
    with open(json_path, "w") as fh:
        fh.write(text + "\n")
    with open(csv_path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
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
