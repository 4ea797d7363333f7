"""Head-width sweep of the FP32 path vs PyTorch FP32 SDPA on the same box:
B1 H16 n (default 16384) at (d, dv) in {64, 128}^2 plus a few odd widths.
Rate = algorithmic 2 n^2 (d + dv) B H / t (the slices' recomputed scores are
overhead, not counted). CUDA events, L2 flushed before every timed call.

usage: python tools/time_wide.py [n] [reps] [d:dv,d:dv,...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23798_b200 as elsa  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
H = 16
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


PAIRS = ((64, 64), (128, 128), (128, 64), (64, 128), (96, 96), (80, 80), (128, 256),
         (256, 256), (256, 64), (192, 192), (32, 32), (16, 16))
if len(sys.argv) > 3:  # explicit "d:dv,d:dv,..."
    PAIRS = tuple(tuple(int(x) for x in p.split(":")) for p in sys.argv[3].split(","))
for d, dv in PAIRS:
    torch.manual_seed(0)
    q = torch.randn(1, H, n, d, device=dev)
    k = torch.randn(1, H, n, d, device=dev)
    v = torch.randn(1, H, n, dv, device=dev)
    fl = 2.0 * n * n * (d + dv) * H
    ms = timeit(lambda: elsa.scaled_dot_product_attention(q, k, v))
    try:
        ms_t = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
        t_s = f"torch SDPA fp32 {ms_t:8.3f} ms {fl / ms_t / 1e9:6.2f} TFLOP/s"
    except RuntimeError as e:  # no fp32 backend for this width
        t_s = f"torch SDPA fp32 n/a ({str(e).splitlines()[0][:60]})"
    print(f"d={d:3d} dv={dv:3d} n={n}: elsa {ms:8.3f} ms {fl / ms / 1e9:6.2f} TFLOP/s | {t_s}",
          flush=True)
    del q, k, v
