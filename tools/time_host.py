"""Host-buffer entry point timing: pinned vs pageable inputs (B1 H16 n16K)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

n, H = 16384, 16
fl = 2.0 * H * n * n * 128
for pinned in (True, False):
    q, k, v = (torch.randn(1, H, n, 64) for _ in range(3))
    out = torch.empty(1, H, n, 64)
    if pinned:
        q, k, v, out = q.pin_memory(), k.pin_memory(), v.pin_memory(), out.pin_memory()
    for _ in range(2):
        elsa.attention_from_host(q, k, v, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        elsa.attention_from_host(q, k, v, out=out)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"{'pinned' if pinned else 'pageable'}: {ms:.2f} ms, {fl / ms / 1e9:.1f} TFLOP/s", flush=True)
