"""Time small shapes several ways: single launch w/ events, back-to-back launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_23798_b200 as elsa
for (b, h, n) in [(1, 16, 1024), (8, 12, 512), (1, 1, 1024), (1, 16, 2048)]:
    q, k, v = (torch.randn(b, h, n, 64, device="cuda") for _ in range(3))
    for _ in range(5):
        elsa.scaled_dot_product_attention(q, k, v)
    torch.cuda.synchronize()
    for splits in (0, 1, 2, 4, 8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        fl = 2 * b * h * n * n * 128
        print(f"B{b} H{h} n{n} splits={splits} ({elsa.describe_plan(q, k, v, splits)}): "
              f"{ms*1e3:.1f} us/call back-to-back, {fl/ms/1e9:.1f} TFLOP/s")
