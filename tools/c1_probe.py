import os, sys
sys.path.insert(0, "/root/repo")
import torch, paper_2604_23798_b200 as elsa
q, k, v = (torch.randn(1, 1, 1024, 64, device="cuda") for _ in range(3))
for s in (0, 4, 16):
    for _ in range(3):
        elsa.scaled_dot_product_attention(q, k, v, kv_splits=s)
torch.cuda.synchronize()
print(elsa.describe_plan(q, k, v))
