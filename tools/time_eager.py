"""Eager (per-call, no CUDA graph) cost of the drop-in for small shapes:
wall time per call over 500 back-to-back calls vs the graph-replayed kernel."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

for (b, h, n) in [(1, 1, 1024), (8, 12, 512), (1, 16, 1024)]:
    q, k, v = (torch.randn(b, h, n, 64, device="cuda") for _ in range(3))
    for _ in range(20):
        elsa.scaled_dot_product_attention(q, k, v)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(500):
        elsa.scaled_dot_product_attention(q, k, v)
    torch.cuda.synchronize()
    us = (time.perf_counter() - t0) / 500 * 1e6
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        elsa.scaled_dot_product_attention(q, k, v)
        with torch.cuda.graph(g, stream=s):
            elsa.scaled_dot_product_attention(q, k, v)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(500):
        g.replay()
    torch.cuda.synchronize()
    gus = (time.perf_counter() - t0) / 500 * 1e6
    print(f"B{b} H{h} n{n}: eager {us:.1f} us/call, graph replay {gus:.1f} us/call", flush=True)
