"""Headline-loop diagnostics: time the B1 H16 n16K forward back to back in
several ways on one box (eager drop-in, eager with out=, CUDA graph, with and
without an L2 flush) to locate differences between the bench's headline and
its graph-replay sweep."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1234)
n = int(os.environ.get("N", "16384"))
q, k, v = (torch.randn(1, 16, n, 64, device=dev, generator=g) for _ in range(3))
fl = 2 * 16 * n * n * 128
s = torch.cuda.current_stream()
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)


def timeit(fn, steps=20, fl_=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


print("plan", elsa.describe_plan(q, k, v))
y0 = torch.empty_like(q)
for rep in range(2):
    ms = timeit(lambda: elsa.scaled_dot_product_attention(q, k, v))
    print(f"eager drop-in        {ms:8.3f} ms  {fl / ms / 1e9:6.2f} TFLOP/s")
    ms = timeit(lambda: elsa.scaled_dot_product_attention(q, k, v, out=y0))
    print(f"eager out=           {ms:8.3f} ms  {fl / ms / 1e9:6.2f} TFLOP/s")

    def fl_step():
        flush.fill_(1.0)
        elsa.scaled_dot_product_attention(q, k, v, out=y0)
    ms_f = timeit(lambda: flush.fill_(1.0))
    ms = timeit(fl_step)
    print(f"eager + flush        {ms - ms_f:8.3f} ms  {fl / (ms - ms_f) / 1e9:6.2f} TFLOP/s (flush {ms_f:.3f})")
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        elsa.scaled_dot_product_attention(q, k, v, out=y0)
    ms = timeit(gr.replay)
    print(f"graph back-to-back   {ms:8.3f} ms  {fl / ms / 1e9:6.2f} TFLOP/s")
    # single launches separated by syncs
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        elsa.scaled_dot_product_attention(q, k, v, out=y0)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        time.sleep(0.05)
    print("isolated launches    " + " ".join(f"{t:.3f}" for t in ts))
