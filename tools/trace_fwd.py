"""Per-warp phase timeline of the forward kernel (needs an ELSA_TRACE build,
loaded through ELSA_LIB_PATH). Prints mean phase durations in ns."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_23798_b200 as elsa
from paper_2604_23798_b200 import _lib

n = int(os.environ.get("N", "16384"))
H = int(os.environ.get("H", "16"))
q, k, v = (torch.randn(1, H, n, 64, device="cuda") for _ in range(3))
for _ in range(3):
    elsa.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
CTAS, WARPS, TILES, PTS = 4, 16, 32, 5
buf = (ctypes.c_ulonglong * (CTAS * WARPS * TILES * PTS))()
h = _lib.lib()
h.elsa_dev_read_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert h.elsa_dev_read_trace(ctypes.cast(buf, ctypes.c_void_p), len(buf)) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(CTAS, WARPS, TILES, PTS)
used = a[..., 0].sum(axis=(0, 2)) > 0
print("warps with data:", np.nonzero(used)[0].tolist())
a = a[:, used]
t0 = a[a > 0].min()
d = np.diff(a, axis=-1)  # wait, gemm1, softmax, gemm2
gap = a[:, :, 1:, 0] - a[:, :, :-1, 4]
valid = (a[..., 0] > 0)
for name, x in (("wait full", d[..., 0]), ("gemm1", d[..., 1]), ("softmax", d[..., 2]),
                ("gemm2", d[..., 3])):
    xs = x[valid]
    print(f"{name:10s} mean {xs.mean():8.0f} ns  p10 {np.percentile(xs,10):8.0f}  p90 {np.percentile(xs,90):8.0f}")
print(f"tile gap   mean {gap[valid[:, :, 1:]].mean():8.0f} ns")
tot = (a[..., 4] - a[..., 0])[valid]
print(f"tile total mean {tot.mean():8.0f} ns")
# warp-to-warp skew at the start of each tile within CTA 0
st = a[0, :, :, 1]
print("CTA0 start skew per tile (ns):", (st.max(axis=0) - st.min(axis=0))[:12].tolist())
print("CTA0 softmax start (rel ns), tile 5:", ((a[0, :, 5, 2] - a[0, :, 5, 1].min())).tolist())
# absolute timeline of CTA 0: kernel-relative first/last marks
print("CTA0 warp0 first mark -> last mark (ns):", int(a[0, 0][a[0, 0] > 0].max() - a[0, 0][a[0, 0] > 0].min()))
