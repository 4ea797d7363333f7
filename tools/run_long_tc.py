"""C5's FP16/BF16 comparison on one GPU: n = 2^20, H = 8, d = 64 through the
tcgen05 variant (K5) and PyTorch's flash SDPA, one timed call each, plus FP64
sampled-row parity of the K5 output. usage: N=1048576 H=8 python tools/run_long_tc.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

n = int(os.environ.get("N", str(1 << 20)))
H = int(os.environ.get("H", "8"))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(7)
fl = 4.0 * H * n * n * 64
for dt in (torch.bfloat16, torch.float16):
    q, k, v = (torch.randn(1, H, n, 64, device=dev, generator=g).to(dt) for _ in range(3))
    for name, fn in (("elsa", lambda: elsa.scaled_dot_product_attention(q, k, v)),
                     ("torch", lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))):
        y = fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{dt} n={n} H={H} {name}: {ms:.1f} ms, {fl / ms / 1e9:.1f} TFLOP/s", flush=True)
        if name == "elsa":
            errs = []
            rng = np.random.default_rng(0)
            for h in (0, H - 1):
                K = k[0, h].double().cpu().numpy()
                V = v[0, h].double().cpu().numpy()
                for r in sorted(set([0, n - 1] + rng.integers(0, n, 6).tolist())):
                    s = (K @ q[0, h, r].double().cpu().numpy()) / math.sqrt(64)
                    s -= s.max()
                    p = np.exp(s)
                    ref = (p @ V) / p.sum()
                    got = y[0, h, r].double().cpu().numpy()
                    errs.append(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
            print(f"  sampled rows {len(errs)}: max rel err {max(errs):.2e} (16-bit output)", flush=True)
    del q, k, v, y
