"""The copy-engine (non-TMA) path vs the TMA path on the same problem: B1 H16
n (default 8192) d = dv = 64 with Q at a 4-byte-aligned offset (4-byte
cp.async), with Q/K/V row-strided 16-byte aligned views (16-byte cp.async:
ELSA_FORCE_GENERIC_LOAD=1 is read once per process, so that leg runs in a
child process), and the TMA path. CUDA events, L2 flushed.

usage: python tools/time_generic.py [n]"""
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23798_b200 as elsa  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fl = 4.0 * 16 * n * n * 64


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


torch.manual_seed(0)
q, k, v = (torch.randn(1, 16, n, 64, device=dev) for _ in range(3))
if os.environ.get("ELSA_FORCE_GENERIC_LOAD"):
    ms = timeit(lambda: elsa.scaled_dot_product_attention(q, k, v))
    print(f"copy engine, 16-byte copies (forced): {ms:8.3f} ms {fl / ms / 1e9:6.2f} TFLOP/s")
    sys.exit(0)
ms = timeit(lambda: elsa.scaled_dot_product_attention(q, k, v))
print(f"TMA:                                  {ms:8.3f} ms {fl / ms / 1e9:6.2f} TFLOP/s")
flat = torch.randn(16 * n * 64 + 1, device=dev)
qm = flat[1:].view(1, 16, n, 64)
ms = timeit(lambda: elsa.scaled_dot_product_attention(qm, k, v))
print(f"copy engine, Q 4-byte aligned:        {ms:8.3f} ms {fl / ms / 1e9:6.2f} TFLOP/s")
subprocess.run([sys.executable, __file__, str(n)], env=dict(os.environ, ELSA_FORCE_GENERIC_LOAD="1"))
