"""`scanattn-bench-v1` records for GPU runs and the paper's
scaling fit. Per-head latency (B = H = 1, as PAPER.md:847-853 measures) for
n = 2^10 .. 2^15 in three modes — scan (FP32 FFMA kernels), scan16 (BF16
tcgen05) and sdpa (PyTorch FP32 SDPA) — then T(n) = a L(n, B) + b n^2 + c per
mode, beside the paper's FP16 A100 fit (a = 0.0142, b = 1.74e-9, c = -0.149,
milliseconds). Writes profiles/<tag>_bench_report.{json,csv}.

usage: python tools/bench_report.py [tag]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_23798_b200 import report  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "round1"
ns = [1 << k for k in range(10, 16)]
records, fits = [], []
for mode in ("scan", "scan16", "sdpa"):
    pts = []
    for n in ns:
        rec = report.run_bench(1, 1, n, mode=mode, repeats=30, warmup=3)
        records.append(rec)
        med = rec.summary()["median"] * 1e3  # seconds -> ms, the paper's unit
        pts.append((n, med))
        print(f"{mode:6s} n={n:6d}: median {med:.4f} ms", flush=True)
    fit = report.fit_scaling(pts, 128)
    fits.append(fit)
    print(f"{mode:6s} fit (ms): a={fit.a:.4g} b={fit.b:.4g} c={fit.c:.4g} "
          f"residual={fit.residual:.3g}", flush=True)
print("paper (FP16, A100, ms): a=0.0142 b=1.74e-9 c=-0.149", flush=True)
jp = os.path.join(ROOT, "profiles", f"{tag}_bench_report.json")
cp = os.path.join(ROOT, "profiles", f"{tag}_bench_report.csv")
report.emit_report(records, fits, jp, cp)
with open(jp) as f:
    doc = json.load(f)
doc["paper_fit_fp16_a100_ms"] = {"a": 0.0142, "b": 1.74e-9, "c": -0.149, "source": "PAPER.md:847-853"}
doc["units"] = "fit coefficients in milliseconds (latencies are stored in seconds per the schema)"
with open(jp, "w") as f:
    json.dump(doc, f, indent=1)
print(jp, cp)
