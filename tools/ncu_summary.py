"""Summarise an `ncu --set full` capture of the forward kernel into
profiles/<tag>.json and profiles/<tag>.md (the numbers bench.py's roofline
`traffic` field and DESIGN.md cite).

usage: python tools/ncu_summary.py <report.ncu-rep> <tag> --b 1 --h 16 --n 16384
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),  # ns -> ms
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "fma_pipe_active_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "smem_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "instructions": ("smsp__inst_executed.sum", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
    "smem_per_block": ("launch__shared_mem_per_block_dynamic", 1.0),
}


def _num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("tag")
    ap.add_argument("--b", type=int, default=1)
    ap.add_argument("--h", type=int, default=16)
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--dv", type=int, default=None, help="V width (default: d)")
    ap.add_argument("--elem-bytes", type=int, default=4, help="4 (FP32) or 2 (FP16/BF16)")
    ap.add_argument("--peak", type=float, default=74.45,
                    help="TFLOP/s denominator: FFMA peak (74.45) for K1, the measured dense "
                         "BF16 peak (MEASURED_PEAKS.json bf16_tflops) for K5")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"report": os.path.basename(a.report), "kernel": d.get("Kernel Name", "")}
    for name, (metric, scale) in KEYS.items():
        v = _num(d.get(metric))
        if v is not None:
            unit = u.get(metric, "")
            if metric.startswith("dram__bytes") and unit in ("Mbyte", "MB"):
                v *= 1e6
            elif metric.startswith("dram__bytes") and unit in ("Gbyte", "GB"):
                v *= 1e9
            elif metric.startswith("dram__bytes") and unit in ("Kbyte", "KB"):
                v *= 1e3
            elif metric == "gpu__time_duration.sum" and unit == "ms":
                scale = 1.0
            elif metric == "gpu__time_duration.sum" and unit == "us":
                scale = 1e-3
            out[name] = v * scale
    stalls = {}
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            x = _num(v)
            if x and x > 0.01:
                stalls[k.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", "")] = round(x, 3)
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    dv = a.d if a.dv is None else a.dv
    flops = 2.0 * a.b * a.h * a.n * a.n * (a.d + dv)
    alg_bytes = float(a.elem_bytes) * a.b * a.h * a.n * (2 * a.d + 2 * dv)
    out["workload"] = f"B{a.b} H{a.h} n{a.n} d{a.d} dv{dv} ({a.elem_bytes}-byte elements)"
    out["algorithmic_flops"] = flops
    out["algorithmic_bytes"] = alg_bytes
    if out.get("dram_read_bytes") is not None:
        out["dram_bytes_per_launch"] = out["dram_read_bytes"] + out.get("dram_write_bytes", 0.0)
        out["traffic_over_algorithmic"] = out["dram_bytes_per_launch"] / alg_bytes
    if out.get("duration_ms"):
        out["tflops_under_ncu"] = flops / (out["duration_ms"] * 1e-3) / 1e12
        out["peak_tflops"] = a.peak
        out["frac_peak_under_ncu"] = out["tflops_under_ncu"] / a.peak
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{a.tag}.json", "w") as f:
        json.dump(out, f, indent=2)
    with open(f"profiles/{a.tag}.md", "w") as f:
        f.write(f"# ncu --set full summary: {a.tag}\n\n")
        f.write(f"Kernel: `{out['kernel']}`  \nWorkload: {out['workload']} "
                f"(algorithmic {flops:.4g} flop, {alg_bytes:.4g} B)\n\n")
        f.write("| metric | value |\n|---|---|\n")
        for k2, v2 in out.items():
            if k2 in ("kernel", "workload", "report", "stalls_per_issue"):
                continue
            f.write(f"| {k2} | {v2:.6g} |\n" if isinstance(v2, float) else f"| {k2} | {v2} |\n")
        f.write("\nWarp stall reasons (per issued instruction):\n\n")
        for k2, v2 in out["stalls_per_issue"].items():
            f.write(f"- {k2}: {v2}\n")
        f.write("\nNumbers taken under the profiler (cold caches, serialised replay) are "
                "evidence for shares and counters, not bench values.\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
