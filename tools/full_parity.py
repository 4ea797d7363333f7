"""Every-row FP64 parity at the headline sizes: the GPU forward (the bench's
path, auto plan) against the FP64 oracle restated from oracles.py:74-104
(row-max-stabilised softmax in float64, numpy on the host), per-row relative
L2 error (verify.py:336-338) against u * L(n, 128) * 8 (verify.py:339-343),
for every query row of every head. usage: python tools/full_parity.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2604_23798_b200 as elsa  # noqa: E402

dev = torch.device("cuda", 0)
shapes = [(1, 16, 16384), (8, 12, 512), (1, 16, 4096), (1, 1, 1024)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
for (B, H, n) in shapes:
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    q, k, v = (torch.randn(B, H, n, 64, device=dev, generator=g) for _ in range(3))
    y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
    torch.cuda.synchronize()
    plan = elsa.describe_plan(q, k, v)
    Y = y.cpu().numpy()
    Q, K, V = (t.cpu().numpy() for t in (q, k, v))
    t0 = time.time()
    errs = []
    for b in range(B):
        for h in range(H):
            ref = oracle.naive_attention_rows_fp64(Q[b:b + 1, h:h + 1], K[b:b + 1, h:h + 1],
                                                   V[b:b + 1, h:h + 1], rows_per_chunk=2048)[0, 0]
            got = Y[b, h].astype(np.float64)
            errs.append(np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1))
    e = np.concatenate(errs)
    thr = oracle.bound_threshold(n)
    print(f"B{B} H{H} n{n} [{plan}]: {e.size} rows, max {e.max():.3e} p99 {np.percentile(e, 99):.3e} "
          f"median {np.median(e):.3e}; bound {thr:.3e}: {'PASS' if e.max() <= thr else 'FAIL'} "
          f"({(e > thr).sum()} rows over; host FP64 {time.time() - t0:.0f} s)", flush=True)
