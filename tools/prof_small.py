"""Small-shape launches for an ncu launch list: each variant runs 5 times
(C1 and friends, cluster merge vs K1 + K2). usage: python tools/prof_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

dev = torch.device("cuda", 0)
shapes = [(1, 1, 1024), (1, 4, 1024), (1, 1, 4096)]
for (b, h, n) in shapes:
    q, k, v = (torch.randn(b, h, n, 64, device=dev) for _ in range(3))
    for mode, s in ((0, 8), (2, 8), (2, 16), (0, 4), (2, 4)):
        elsa.attention.set_cluster_mode(mode)
        print(f"B{b} H{h} n{n} mode {mode} splits {s}: {elsa.describe_plan(q, k, v, s)}", flush=True)
        for _ in range(5):
            elsa.scaled_dot_product_attention(q, k, v, kv_splits=s)
        torch.cuda.synchronize()
elsa.attention.set_cluster_mode(1)
