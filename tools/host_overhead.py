"""Where the eager (no CUDA graph) per-call host time of the drop-in goes, for
small shapes: the whole call vs its parts, each timed over N back-to-back
calls with the GPU work kept trivially short. usage: python tools/host_overhead.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402
from paper_2604_23798_b200 import _lib, attention as att  # noqa: E402

N = 2000
dev = torch.device("cuda", 0)


def per_call(fn, n=N):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


for (b, h, n) in [(1, 1, 1024), (8, 12, 512), (1, 1, 64)]:
    q, k, v = (torch.randn(b, h, n, 64, device=dev) for _ in range(3))
    y = torch.empty_like(q)
    lib = _lib.lib()
    shp = att._shape(q, k, v, y)
    ws_bytes = lib.elsa_workspace_bytes(ctypes.byref(shp), 0)
    ws = torch.empty(max(ws_bytes, 1), device=dev, dtype=torch.uint8)
    stream = att._stream_ptr(dev)
    args = (ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.byref(shp),
            ctypes.c_double(0.125), 0, ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws_bytes),
            stream)
    rows = {
        "eager drop-in": per_call(lambda: elsa.scaled_dot_product_attention(q, k, v)),
        "drop-in, out=": per_call(lambda: elsa.scaled_dot_product_attention(q, k, v, out=y)),
        "ctypes elsa_fwd_f32 only": per_call(lambda: lib.elsa_fwd_f32(*args)),
        "ctypes resolve_kv_splits (plan)": per_call(
            lambda: lib.elsa_resolve_kv_splits(ctypes.byref(shp), 0)),
        "torch.empty(workspace)": per_call(
            lambda: torch.empty(max(ws_bytes, 1), device=dev, dtype=torch.uint8)),
        "torch.empty(Y)": per_call(lambda: torch.empty((b, h, n, 64), device=dev)),
        "python checks (_validate/_as_4d/_prep)": per_call(
            lambda: [att._validate(q, k, v, True)] + [att._prep(att._as_4d(t, "x")) for t in (q, k, v)]),
        "current_stream ptr": per_call(lambda: att._stream_ptr(dev)),
        "torch.cuda.device ctx": per_call(lambda: torch.cuda.device(dev).__enter__()),
    }
    print(f"B{b} H{h} n{n} plan [{elsa.describe_plan(q, k, v)}] ws={ws_bytes}")
    for kk, vv in rows.items():
        print(f"   {kk:42s} {vv:7.2f} us/call", flush=True)
