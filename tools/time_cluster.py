"""Cluster split merge (K1 CL = true) vs the two-launch split path (K1 + K2)
vs one split: CUDA-graph replays with the L2 flushed between them (the bench
sweep's protocol), per shape and split count. usage: python tools/time_cluster.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402
from paper_2604_23798_b200 import _lib  # noqa: E402

h = _lib.lib()
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream(dev)


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs[2:]])) * 1e3


shapes = [(1, 1, 1024), (8, 12, 512), (1, 16, 1024), (1, 16, 2048), (1, 16, 4096),
          (1, 4, 1024), (2, 16, 512), (1, 1, 4096), (1, 1, 16384)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
CFG = os.environ.get("CFG")  # force a configuration (e.g. w8r4) for the split rows
for (b, hh, n) in shapes:
    q, k, v = (torch.randn(b, hh, n, 64, device=dev) for _ in range(3))
    y_ref = elsa.scaled_dot_product_attention(q, k, v)
    fl = 2.0 * b * hh * n * n * 128
    elsa.attention.set_cluster_mode(1)
    elsa.attention.force_config(None)
    auto = elsa.describe_plan(q, k, v)
    t_auto = timed(lambda: elsa.scaled_dot_product_attention(q, k, v))
    print(f"B{b} H{hh} n{n}: auto [{auto}] {t_auto:.1f} us {fl / t_auto / 1e6:.1f} TFLOP/s",
          flush=True)
    if CFG:
        elsa.attention.force_config(CFG)
    for s in (1, 2, 4, 8, 16):
        row = []
        for mode in (0, 2):
            elsa.attention.set_cluster_mode(mode)
            plan = elsa.describe_plan(q, k, v, s)
            dy = (elsa.scaled_dot_product_attention(q, k, v, kv_splits=s) - y_ref).abs().max().item()
            assert dy < 1e-4, (plan, dy)
            t = timed(lambda: elsa.scaled_dot_product_attention(q, k, v, kv_splits=s))
            row.append(f"{'clu' if 'cluster' in plan else 'k2 '} {t:7.1f} us ({plan.split()[0]})")
        print(f"   splits {s:2d}: " + " | ".join(row), flush=True)
    elsa.attention.set_cluster_mode(1)
    elsa.attention.force_config(None)
