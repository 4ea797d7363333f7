"""Per-tile timeline of K5 in CTA 0 (build: tools/variant_sweep.sh
"tctrace:-DELSA_TC_TRACE", run with ELSA_LIB_PATH=build/var_tctrace.so).
Softmax warp points: 0 before s_full wait, 1 S ready, 2 s_free arrived,
3 row max done, 4 O rescaled (anchor moves only), 5 p_full arrived. MMA slots 8+g: 0 S issue,
1 PV issue. Prints SM clocks relative to the first stamp."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402
from paper_2604_23798_b200 import _lib  # noqa: E402

T = 64
n = int(os.environ.get("N", "16384"))
q, k, v = (torch.randn(1, 16, n, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(2):
    elsa.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (16 * T * 8))()
h = _lib.lib()
h.elsa_dev_read_tc_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert h.elsa_dev_read_tc_trace(ctypes.cast(buf, ctypes.c_void_p), 16 * T * 8) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(16, T, 8).astype(np.int64)
t0 = a[a > 0].min()
a = np.where(a > 0, a - t0, -1)
for t in range(8, 40):
    sm = [a[w, t] for w in (0, 4)]
    mma = [a[8 + g, t] for g in (0, 1)]
    print(f"t{t:3d} g0 {list(sm[0][:6])} g1 {list(sm[1][:6])} | S/PV issue g0 {list(mma[0][:2])} g1 {list(mma[1][:2])}")
# averages over tiles 8..56: durations
d = lambda w, x, y: np.mean([a[w, t, y] - a[w, t, x] for t in range(8, 56)])
for w in (0, 1, 4):
    print(f"warp {w}: wait S {d(w,0,1):7.0f}  ld S {d(w,1,2):6.0f}  max {d(w,2,3):6.0f}  "
          f"exp/P (incl. O wait) {d(w,3,5):6.0f}  tile {np.mean(np.diff(a[w, 8:56, 0])):7.0f} clk")
print("S issue -> S ready (g0):", np.mean([a[0, t, 1] - a[8, t, 0] for t in range(8, 56)]))
print("p_full -> PV issue (g0):", np.mean([a[8, t, 1] - a[0, t, 5] for t in range(8, 56)]))
print("s_free -> S issue (g0):", np.mean([a[8, t + 1, 0] - a[0, t, 2] for t in range(8, 56)]))
print("O wait before the first P store (warp 0, warp 4):",
      np.mean([a[0, t, 7] - a[0, t, 6] for t in range(8, 56)]),
      np.mean([a[4, t, 7] - a[4, t, 6] for t in range(8, 56)]),
      "| max done -> O wait start:", np.mean([a[0, t, 6] - a[0, t, 3] for t in range(8, 56)]))
print("S issue call duration (g0):", np.mean([a[8, t, 2] - a[8, t, 0] for t in range(8, 56)]))
print("PV issue call duration (g0):", np.mean([a[8, t, 3] - a[8, t, 1] for t in range(8, 56)]))
ev = sorted([(a[8 + g, t, k], f"{'S' if k == 0 else 'PV'}{g}({t})", a[8 + g, t, k + 2] - a[8 + g, t, k])
             for g in (0, 1) for t in range(30, 40) for k in (0, 1)])
print("MMA warp issue sequence (clk, event, call duration):")
for e in ev:
    print("  ", e)
