"""A/B timing of libelsa builds: python tools/ab_time.py [tag] — times the
forward on a fixed shape list (CUDA-graph replays, L2 flushed between,
events on the replay stream) with the library ELSA_LIB_PATH points at, and
prints one line per shape. Run once per build, alternating, on one box."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

SHAPES = [(1, 16, 1024), (1, 16, 2048), (1, 16, 4096), (1, 16, 8192), (1, 16, 16384),
          (8, 12, 512), (1, 1, 1024)]
if os.environ.get("AB_SHAPES"):
    SHAPES = [tuple(int(x) for x in s.split("x")) for s in os.environ["AB_SHAPES"].split(",")]
tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("ELSA_LIB_PATH", "default")
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream(dev)
for (b, h, n) in SHAPES:
    q, k, v = (torch.randn(b, h, n, 64, device=dev) for _ in range(3))
    with torch.cuda.stream(s):
        for _ in range(3):
            elsa.scaled_dot_product_attention(q, k, v)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            elsa.scaled_dot_product_attention(q, k, v)
        torch.cuda.synchronize()
        reps = 40 if n <= 4096 else 10
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            z = torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            z.record(s)
            ts.append((a, z))
        torch.cuda.synchronize()
    t = sorted(x.elapsed_time(y) for x, y in ts[2:])
    ms = t[len(t) // 2]
    fl = 2.0 * b * h * n * n * 128
    print(f"{tag:10s} B{b} H{h} n{n:6d}: {ms*1e3:9.1f} us {fl/ms/1e9:6.1f} TF/s  "
          f"({elsa.describe_plan(q, k, v)})", flush=True)
    del g
