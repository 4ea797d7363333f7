"""One-off long-context run on one GPU: n = 2^20 (C5, H = 8) or 64K (C4),
timed forward + FP64 sampled-row parity. usage: N=1048576 H=8 python tools/run_long.py"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_2604_23798_b200 as elsa
n = int(os.environ.get("N", str(1 << 20)))
H = int(os.environ.get("H", "8"))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(7)
q, k, v = (torch.randn(1, H, n, 64, device=dev, generator=g) for _ in range(3))
print("plan:", elsa.describe_plan(q, k, v), flush=True)
y = elsa.scaled_dot_product_attention(q, k, v)  # warm-up (also the parity sample)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
fl = 2.0 * H * n * n * 128
print(f"n={n} H={H}: {ms:.1f} ms, {fl / ms / 1e9:.2f} TFLOP/s, {fl / ms / 1e9 / 74.45:.3f} of FFMA peak", flush=True)
rng = np.random.default_rng(0)
errs = []
for h in (0, H - 1):
    K = k[0, h].double().cpu().numpy()
    V = v[0, h].double().cpu().numpy()
    for r in sorted(set([0, n - 1] + rng.integers(0, n, 6).tolist())):
        qv = q[0, h, r].double().cpu().numpy()
        s = (K @ qv) / math.sqrt(64)
        s -= s.max()
        p = np.exp(s)
        ref = (p @ V) / p.sum()
        got = y[0, h, r].double().cpu().numpy()
        errs.append(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
thr = oracle.bound_threshold(n)
print(f"sampled rows {len(errs)}: max rel err {max(errs):.3e}, bound u*L(n,128)*8 = {thr:.3e}, "
      f"{'PASS' if max(errs) <= thr else 'FAIL'}", flush=True)
