"""Kernel time of (config, kv_splits) for small shapes: median of single
launches bracketed by CUDA events, L2 flushed in between. Config is forced via
ELSA_FWD_CFG in the environment of this process."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_23798_b200 as elsa
flush = torch.empty(64 * 1024 * 1024, device="cuda")
# bring SM clocks up (the part idles at ~120 MHz): ~200 ms of dense work
_w = torch.randn(8192, 8192, device="cuda")
for _ in range(40):
    _w = _w @ _w.T * 1e-4
torch.cuda.synchronize()
shapes = [(1, 16, 1024), (8, 12, 512), (1, 1, 1024), (1, 16, 2048), (1, 16, 4096)]
if os.environ.get("PLAN_SHAPES"):
    shapes = [tuple(int(x) for x in s.split("x")) for s in os.environ["PLAN_SHAPES"].split(",")]
for (b, h, n) in shapes:
    q, k, v = (torch.randn(b, h, n, 64, device="cuda") for _ in range(3))
    for splits in (1, 2, 3, 4, 6, 8, 16):
        if splits > n // 64:
            continue
        for _ in range(3):
            elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits)
        torch.cuda.synchronize()
        # time a captured CUDA graph so host-side Python overhead is excluded
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits)
        torch.cuda.synchronize()
        evs = []
        for _ in range(30):  # back-to-back: flush, event, graph, event (no host idle gaps)
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) for a, b in evs[5:]]
        ms = float(np.median(ts))
        fl = 2 * b * h * n * n * 128
        print(f"{os.environ.get('ELSA_FWD_CFG','auto'):6s} B{b} H{h} n{n} s={splits:2d}: {ms*1e3:7.1f} us "
              f"{fl/ms/1e9:5.1f} TF/s  [{elsa.describe_plan(q, k, v, splits)}]", flush=True)
