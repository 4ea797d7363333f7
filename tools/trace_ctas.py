"""CTA start/end timeline of one forward launch (ELSA_TRACE build via ELSA_LIB_PATH)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_23798_b200 as elsa
from paper_2604_23798_b200 import _lib
B, H, n = (int(x) for x in os.environ.get("SHAPE", "1,16,1024").split(","))
splits = int(os.environ.get("SPLITS", "0"))
q, k, v = (torch.randn(B, H, n, 64, device="cuda") for _ in range(3))
for _ in range(3):
    elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits)
torch.cuda.synchronize()
h = _lib.lib()
h.elsa_dev_read_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
W0 = 4 * 16 * 32 * 5
tot = W0 + 3 * 8192
buf = (ctypes.c_ulonglong * tot)()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits)
e1.record()
torch.cuda.synchronize()
assert h.elsa_dev_read_trace(ctypes.cast(buf, ctypes.c_void_p), tot) == 0
a = np.frombuffer(buf, dtype=np.uint64)[W0:].reshape(-1, 3).astype(np.int64)
plan = elsa.describe_plan(q, k, v, splits)
ncta = int((a[:, 0] > 0).sum())
a = a[:ncta]
t0 = a[:, 0].min()
st, en, sm = a[:, 0] - t0, a[:, 1] - t0, a[:, 2]
print(plan, "ctas", ncta, "event ms", e0.elapsed_time(e1))
print(f"start: min 0 max {st.max()} ns; end: min {en.min()} median {np.median(en):.0f} max {en.max()} ns")
dur = en - st
print(f"CTA duration: min {dur.min()} median {np.median(dur):.0f} max {dur.max()} ns")
per_sm = np.bincount(sm, minlength=148)
print("CTAs per SM histogram:", np.bincount(per_sm).tolist())
# per-warp tile marks for CTAs 0..3 relative to each CTA's start
wm = np.frombuffer(buf, dtype=np.uint64)[:W0].reshape(4, 16, 32, 5).astype(np.int64)
for c in range(min(4, ncta)):
    s0 = a[c, 0]
    w = wm[c]
    used = (w[:, :, 0] > 0).any(axis=1)
    w = w[used]
    first = w[:, 0, 0].min() - s0
    last = w[:, :, 4][w[:, :, 4] > 0].max() - s0
    print(f"CTA{c} (SM {a[c,2]}): first tile mark +{first} ns, last tile end +{last} ns, CTA end +{a[c,1]-s0} ns, "
          f"tiles/warp {int((w[0, :, 0] > 0).sum())}, mean tile {np.mean(w[:, :, 4][w[:, :, 4] > 0] - w[:, :, 0][w[:, :, 4] > 0]):.0f} ns")
    print("   per-tile total (warp0):", (w[0, :, 4] - w[0, :, 0])[:16].tolist())
    nt = int((w[0, :, 4] > 0).sum())
    if nt < w.shape[1]:
        e = w[:, nt, :3] - s0
        print("   epilogue marks (start, after normalizers, end) per warp:", e.tolist())
