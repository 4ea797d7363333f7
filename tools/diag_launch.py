import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_23798_b200 as elsa
q = torch.randn(1, 2, 512, 64, device="cuda")
try:
    y = elsa.scaled_dot_product_attention(q, q, q)
    torch.cuda.synchronize()
    print("ok", os.environ.get("ELSA_FWD_CFG"))
except Exception as e:
    print("fail", os.environ.get("ELSA_FWD_CFG"), e)
