"""Run the forward kernel a few times on one config (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=1)
ap.add_argument("--h", type=int, default=16)
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--splits", type=int, default=0)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--dv", type=int, default=64)
a = ap.parse_args()
dev = torch.device("cuda", 0)
q, k = (torch.randn(a.b, a.h, a.n, a.d, device=dev) for _ in range(2))
v = torch.randn(a.b, a.h, a.n, a.dv, device=dev)
for _ in range(a.reps):
    elsa.scaled_dot_product_attention(q, k, v, kv_splits=a.splits)
torch.cuda.synchronize()
print("done")
