"""Golden fixtures for the block-level rows of SURVEY §8(f): block totals
and exclusive prefixes (engine.inter_block_combine / blockwise_states), the
ATN1 tensor file format (tensorio.write_tensor) and the bench report schema
and scaling fit (bench.BenchRecord / fit_scaling / emit_report).

Run in the build container (where /root/reference exists, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_blocks.py

Writes tests/golden/blocks.npz and tests/golden/harness.npz. Nothing at test
time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import scanattn as sa
    from scanattn import engine, bench, tensorio, verify

    blk = {}
    rng = np.random.default_rng(23798)
    # ---- inter_block_combine totals + exclusive prefixes (engine.py:265-297) ----
    for dt, prec in ((np.float32, sa.Precision.FP32), (np.float64, sa.Precision.FP64)):
        tag = "f32" if dt == np.float32 else "f64"
        for K in (1, 2, 3, 5, 8, 9, 13, 32):
            ts = []
            for i in range(K):
                if K >= 5 and i in (1, K - 2):
                    ts.append(sa.identity(6, prec))
                else:
                    ts.append(sa.StateTriple(dt(rng.uniform(-30, 30)), dt(rng.uniform(0.5, 9)),
                                             rng.standard_normal(6).astype(dt)))
            total, pre = engine.inter_block_combine(ts, return_prefixes=True)
            blk[f"ibc_{tag}_{K}_in"] = np.stack([np.concatenate([[t.m, t.S], t.W]) for t in ts])
            blk[f"ibc_{tag}_{K}_total"] = np.concatenate([[total.m, total.S], total.W])
            blk[f"ibc_{tag}_{K}_pre"] = np.stack([np.concatenate([[t.m, t.S], t.W]) for t in pre])

    # ---- blockwise_states (engine.py:430-451) on a seeded FP32 problem ----
    spec = dict(seed=11, scenario="regular", b=1, h=2, n=100, d=16, d_v=8)
    p32 = sa.generate(sa.GeneratorSpec(precision=sa.Precision.FP32, **spec))
    cfg = sa.ScanConfig(block_size=128, precision=sa.Precision.FP32)
    blk["bw_spec"] = np.array([spec["seed"], spec["b"], spec["h"], spec["n"], spec["d"],
                               spec["d_v"]])
    for B in (7, 32, 64, 128):
        for hi in (0, 1):
            for qi in (0, 33, 99):
                st = engine.blockwise_states(p32, cfg, qi, b_idx=0, h_idx=hi, block_size=B)
                blk[f"bw_{B}_{hi}_{qi}"] = np.stack([np.concatenate([[t.m, t.S], t.W]) for t in st])
    rep = verify.block_validation(p32, cfg, [7, 32, 128])
    blk["bv_devs"] = np.array([rep.max_pairwise_dev, rep.max_vs_sequential_dev])
    np.savez_compressed(os.path.join(OUT, "blocks.npz"), **blk)

    # ---- ATN1 (tensorio.py:198-239) and the bench report (bench.py:40-242) ----
    har = {}
    with tempfile.TemporaryDirectory() as tmp:
        for tag, prec in (("f32", sa.Precision.FP32), ("f64", sa.Precision.FP64)):
            p = sa.generate(sa.GeneratorSpec(seed=5, scenario="regular", b=1, h=2, n=3, d=4,
                                             d_v=4, precision=prec))
            path = os.path.join(tmp, f"{tag}.atn")
            tensorio.write_tensor(path, p.Q)
            with open(path, "rb") as f:
                har[f"atn1_{tag}_bytes"] = np.frombuffer(f.read(), dtype=np.uint8)
            har[f"atn1_{tag}_data"] = p.Q.data
        rec = bench.BenchRecord(mode="scan", n=1024, block_size=128, tile_q=64, d=64, d_v=64,
                                b=1, h=16, precision="fp32", repeats=5, warmup=2,
                                latencies=[3.0e-4, 2.5e-4, 2.7e-4, 2.6e-4, 2.9e-4],
                                merge_count=123, leaf_count=456, peak_extra_memory=789)
        pts = [(1024, 1.1e-4), (2048, 3.9e-4), (4096, 1.5e-3), (8192, 5.6e-3), (16384, 2.2e-2)]
        fit = bench.fit_scaling(pts, 128)
        jp, cp = bench.emit_report([rec], [fit], os.path.join(tmp, "r.json"))
        with open(jp) as f:
            har["report_json"] = np.frombuffer(f.read().encode(), dtype=np.uint8)
        with open(cp) as f:
            har["report_csv"] = np.frombuffer(f.read().encode(), dtype=np.uint8)
        har["fit_pts"] = np.array(pts)
        har["fit_coef"] = np.array([fit.a, fit.b, fit.c, fit.residual])
        har["pct_in"] = rng.standard_normal(101)
        pc = verify.nearest_rank_percentiles(har["pct_in"])
        har["pct_out"] = np.array([pc["median"], pc["p95"], pc["p99"]])
    np.savez_compressed(os.path.join(OUT, "harness.npz"), **har)
    print("wrote blocks.npz, harness.npz;", json.dumps({"bv": blk["bv_devs"].tolist()}))


if __name__ == "__main__":
    main()
