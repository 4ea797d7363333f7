"""Print the planner's choice for shapes without a GPU (the C-ABI planner
falls back to 148 SMs when no device is present).
usage: python tools/plan_cpu.py B,H,n[,d,dv] ..."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_23798_b200 import _lib  # noqa: E402

h = _lib.lib()
for arg in sys.argv[1:] or ["1,16,16384", "1,16,65536", "1,8,1048576", "8,12,512", "1,1,1024"]:
    vals = [int(x) for x in arg.split(",")]
    B, H, n = vals[:3]
    d = vals[3] if len(vals) > 3 else 64
    dv = vals[4] if len(vals) > 4 else d
    s = _lib.ElsaShape()
    s.B, s.H, s.n_q, s.n_kv, s.d, s.dv = B, H, n, n, d, dv
    for name, w in (("q_stride", d), ("k_stride", d), ("v_stride", dv), ("y_stride", dv)):
        st = getattr(s, name)
        st[0], st[1], st[2] = H * n * w, n * w, w
    buf = ctypes.create_string_buffer(256)
    rc = h.elsa_describe_plan(ctypes.byref(s), 0, buf, 256)
    print(f"B{B} H{H} n{n} d{d} dv{dv}: rc={rc} {buf.value.decode()}")
