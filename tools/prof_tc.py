"""Run the FP16/BF16 tcgen05 forward a few times (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

n = int(os.environ.get("N", "16384"))
dt = torch.bfloat16 if os.environ.get("DT", "bf16") == "bf16" else torch.float16
q, k, v = (torch.randn(1, 16, n, 64, device="cuda", dtype=dt) for _ in range(3))
for _ in range(3):
    elsa.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
print("done")
