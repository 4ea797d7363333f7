"""Per-kernel SASS opcode counts of libelsa.so (fwd_f32_kernel instantiations
by default) and an opcode-sequence fingerprint, to check that a source change
left a tuned kernel's instruction stream alone.

usage: python tools/sass_stats.py [lib.so] [name-filter] [--dump DIR]"""
import hashlib
import os
import re
import subprocess
import sys
from collections import Counter

args = [a for a in sys.argv[1:] if not a.startswith("--")]
lib = args[0] if args else os.path.join(os.path.dirname(__file__), "..", "paper_2604_23798_b200", "libelsa.so")
flt = args[1] if len(args) > 1 else "fwd_f32_kernel"
dump = sys.argv[sys.argv.index("--dump") + 1] if "--dump" in sys.argv else None
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    if flt not in name:
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,6}\*/\s+([^;]*);", f)
    ops = [(i.split()[1] if i.startswith("@") else i.split()[0]) for i in ins]
    c = Counter(o.split(".")[0] for o in ops)
    fp = hashlib.sha1("\n".join(ins).encode()).hexdigest()[:12]
    keys = ("FFMA2", "FFMA", "LDS", "STS", "MUFU", "BRA", "SHFL")
    print(f"{name[:100]} n={len(ins)} fp={fp} " + " ".join(f"{k}={c[k]}" for k in keys))
    if dump:
        os.makedirs(dump, exist_ok=True)
        with open(os.path.join(dump, hashlib.sha1(name.encode()).hexdigest()[:10] + ".sass"), "w") as fh:
            fh.write(name + "\n" + "\n".join(ins) + "\n")
