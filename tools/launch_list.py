"""Turn an `ncu --metrics gpu__time_duration.sum --csv` launch list into
profiles/<tag>_launches.md (per-launch table + share of the forward kernel).

usage: python tools/launch_list.py <launches.csv> <tag> [command description]"""
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main():
    path, tag = sys.argv[1], sys.argv[2]
    cmd = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    bi = h.index("Block Size") if "Block Size" in h else None
    launches = []
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        ms = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-6)
        launches.append((r[ki], r[gi] if gi is not None else "", r[bi] if bi is not None else "", ms))
    total = sum(x[3] for x in launches)
    fwd = sum(x[3] for x in launches if "fwd_f32_kernel" in x[0])
    ours = sum(x[3] for x in launches if "elsa::" in x[0])
    out = [f"# Launch list: {cmd or tag}", "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold "
           "caches: shares, not bench values)", "",
           "| # | kernel | grid | block | ms | share |", "|---|---|---|---|---|---|"]
    for i, (k, g, b, ms) in enumerate(launches):
        name = k.split("(")[0][:70]
        out.append(f"| {i} | `{name}` | {g} | {b} | {ms:.3f} | {100 * ms / total:.1f}% |")
    out += ["", f"Total {total:.3f} ms; elsa kernels {ours:.3f} ms ({100 * ours / total:.1f}%); "
                f"forward kernel {fwd:.3f} ms ({100 * fwd / total:.1f}%)."]
    dst = os.path.join(ROOT, "profiles", f"{tag}_launches.md")
    with open(dst, "w") as f:
        f.write("\n".join(out) + "\n")
    print(dst)


if __name__ == "__main__":
    main()
