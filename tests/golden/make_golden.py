"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package ``scanattn`` from
/root/reference/pkg/src and records its outputs for small, seeded cases:
generator tensors (tensorio.generate), the depth table (engine.scan_depth),
monoid merges and trees (monoid.merge_lanes / merge_tree / merge), FP64
naive attention (oracles.naive_attention), the reference's FP32 blocked scan
(engine.scan_forward) and bound-check thresholds (verify.bound_check). The
fixtures travel with the repo; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import scanattn as sa

    # ---- generator (tensorio.py:125-195) ----
    gen = {}
    specs = [
        ("g0", dict(seed=11, scenario="regular", b=1, h=1, n=64, d=16, d_v=8, precision=sa.Precision.FP32)),
        ("g1", dict(seed=13, scenario="stress", b=1, h=2, n=32, d=8, d_v=8, precision=sa.Precision.FP64)),
        ("g2", dict(seed=0, scenario="regular", b=2, h=2, n=16, d=64, d_v=64, precision=sa.Precision.FP32)),
        ("g3", dict(seed=107, scenario="long", b=1, h=1, n=24, d=8, d_v=8, precision=sa.Precision.FP32)),
    ]
    for tag, kw in specs:
        p = sa.generate(sa.GeneratorSpec(**kw))
        gen[f"{tag}_Q"], gen[f"{tag}_K"], gen[f"{tag}_V"] = p.Q.data, p.K.data, p.V.data
        gen[f"{tag}_spec"] = np.array([kw["seed"], kw["b"], kw["h"], kw["n"], kw["d"], kw["d_v"],
                                       ["regular", "long", "stress"].index(kw["scenario"]),
                                       32 if kw["precision"] is sa.Precision.FP32 else 64])
    np.savez_compressed(os.path.join(OUT, "generator.npz"), **gen)

    # ---- depth table (engine.py:47-55; test_engine.py:40-50) ----
    pts = [(1, 1), (64, 128), (100, 16), (128, 128), (256, 128), (512, 128), (1024, 128),
           (2048, 128), (4096, 128), (8192, 128), (16384, 128), (65536, 128), (1 << 20, 128),
           (300, 32), (1000, 7)]
    np.savez_compressed(os.path.join(OUT, "depth.npz"),
                        pts=np.array(pts), depth=np.array([sa.scan_depth(n, b) for n, b in pts]),
                        cap=np.array([sa.depth_cap(n) for n, _ in pts]))

    # ---- monoid (monoid.py:160-265) ----
    mon = {}
    rng = np.random.default_rng(2604)
    for dt in (np.float64, np.float32):
        k = 64
        ma, mb = rng.uniform(-20, 20, (2, k)).astype(dt)
        mb[:8] = ma[:8]                       # ties
        ma[8:12] = -np.inf                    # identity operands
        mb[10:14] = -np.inf                   # incl. identity (+) identity at 10, 11
        Sa, Sb = rng.uniform(0, 5, (2, k)).astype(dt)
        Wa, Wb = rng.standard_normal((2, k, 3)).astype(dt)
        Sa[ma == -np.inf] = 0
        Wa[ma == -np.inf] = 0
        Sb[mb == -np.inf] = 0
        Wb[mb == -np.inf] = 0
        m, S, W = sa.merge_lanes(ma, Sa, Wa, mb, Sb, Wb)
        tag = "f64" if dt == np.float64 else "f32"
        for name, arr in (("ma", ma), ("Sa", Sa), ("Wa", Wa), ("mb", mb), ("Sb", Sb), ("Wb", Wb),
                          ("m", m), ("S", S), ("W", W)):
            mon[f"lanes_{tag}_{name}"] = arr
        for cnt in range(1, 10):
            ts = [sa.StateTriple(dt(rng.uniform(-20, 20)), dt(rng.uniform(0, 5)),
                                 rng.standard_normal(4).astype(dt)) for _ in range(cnt)]
            if cnt >= 4:
                ts[1] = sa.identity(4, sa.Precision.FP32 if dt == np.float32 else sa.Precision.FP64)
            out = sa.merge_tree(ts)
            mon[f"tree_{tag}_{cnt}_m"] = np.array([t.m for t in ts], dtype=dt)
            mon[f"tree_{tag}_{cnt}_S"] = np.array([t.S for t in ts], dtype=dt)
            mon[f"tree_{tag}_{cnt}_W"] = np.stack([t.W for t in ts]).astype(dt)
            mon[f"tree_{tag}_{cnt}_out"] = np.concatenate([[out.m, out.S], out.W]).astype(dt)
    ln2 = np.log(2.0)
    kat = sa.merge(sa.StateTriple(ln2, 1.0, np.array([1.0])), sa.StateTriple(0.0, 1.0, np.array([1.0])))
    mon["kat_ln2"] = np.array([kat.m, kat.S, kat.W[0]])
    kat = sa.merge(sa.StateTriple(0.0, 1.0, np.array([1.0])), sa.StateTriple(0.0, 1.0, np.array([3.0])))
    mon["kat_equal"] = np.array([kat.m, kat.S, kat.W[0]])
    np.savez_compressed(os.path.join(OUT, "monoid.npz"), **mon)

    # ---- attention outputs: FP64 naive and the reference FP32 scan ----
    att = {}
    cases = [
        ("a0", dict(seed=11, scenario="regular", b=1, h=1, n=256, d=16, d_v=8)),
        ("a1", dict(seed=13, scenario="stress", b=1, h=2, n=128, d=32, d_v=32)),
        ("a2", dict(seed=0, scenario="regular", b=1, h=2, n=200, d=64, d_v=64)),
        ("a3", dict(seed=0, scenario="regular", b=1, h=1, n=1, d=4, d_v=4)),
        ("a4", dict(seed=107, scenario="long", b=1, h=1, n=130, d=8, d_v=8)),
    ]
    for tag, kw in cases:
        p32 = sa.generate(sa.GeneratorSpec(precision=sa.Precision.FP32, **kw))
        ref = sa.naive_attention(p32, sa.Precision.FP64)
        out, _ = sa.scan_forward(p32, sa.ScanConfig(block_size=128, tile_q=64,
                                                    precision=sa.Precision.FP32))
        rep = sa.bound_check(p32, sa.ScanConfig(block_size=128, precision=sa.Precision.FP32),
                             candidate=out, reference=ref)
        att[f"{tag}_spec"] = np.array([kw["seed"], kw["b"], kw["h"], kw["n"], kw["d"], kw["d_v"],
                                       ["regular", "long", "stress"].index(kw["scenario"])])
        att[f"{tag}_y64"] = ref.Y.data
        att[f"{tag}_scan32"] = out.Y.data
        att[f"{tag}_bound"] = np.array([rep.depth, rep.threshold, rep.max_row_error,
                                        float(rep.rows_failed)])
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **att)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
