#!/usr/bin/env python
"""ELSA FP32 exact attention on B200 — the driver's benchmark.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl elsa|reference]

Workload (BASELINE.json configs[2], the config its metric is quoted on):
FP32 attention B=1 H=16 d=dv=64 at n=16384 — one "step" is one full forward
over the (B, H, n, d) problem. The headline `value` is whole-job TFLOP/s with
algorithmic flops 2*B*H*n^2*(d+dv) (QK^T + PV, FMA = 2; exps not counted),
inputs resident in HBM (3 x 67 MB > the 126 MB L2, so consecutive steps do not
hit in L2). `e2e` is the same metric through the public drop-in
(`paper_2604_23798_b200.attention_from_host` -> C-ABI `elsa_fwd_f32_host`)
with pinned host buffers: H2D of Q/K/V and D2H of Y inside the timed region,
pipelined per head group under the kernels. The 1K..16K sweep
(plus BERT-base and the single-head config) is reported beside it with the
L2 flushed between timed iterations.

N > 1 (torchrun, one rank per GPU, NCCL): the same problem KV-sharded across
the ranks (paper_2604_23798_b200.dist: per-chunk (m,S,W) states, one
all_to_all, fixed (+)-tree merge) — strong scaling of a fixed problem.

`--impl reference` times the reference's own CPU algorithm (the blocked
scan of scanattn.engine.scan_forward, restated bit-exactly in
oracle/scan_port.py) on the host cores, on a bounded sample of the same
workload (whole 64-query tiles), and reports the same metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("FP32 attention ms & TFLOP/s vs seq len 1K–16K; % of FP32 FFMA peak; "
          "1/2/4/8 GPU")
SMS = 148
FFMA_LANES = 128


def flops(b, h, n_q, n_kv, d=64, dv=64):
    return 2.0 * b * h * n_q * n_kv * (d + dv)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["elsa", "reference"], default="elsa")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-tiles", type=int, default=0,
                    help="64-query tiles per CPU sample (0 = one per worker)")
    ap.add_argument("--cpu-workers", type=int, default=0)
    ap.add_argument("--dist-path", action="store_true",
                    help="run the KV-sharded multi-GPU code path even at N = 1 (a world-size-1 "
                         "NCCL group; checks the N > 1 path on a single GPU)")
    ap.add_argument("--shard", choices=["kv", "q"], default="kv",
                    help="N > 1: KV-sharded (Proposition 1, the product) or query-sharded "
                         "(no exchange; SURVEY 8e's control experiment)")
    ap.add_argument("--exchange", choices=["peer", "nccl"], default="peer",
                    help="N > 1: state exchange + merge over symmetric peer memory (one "
                         "kernel) or NCCL all_to_all + merge kernel")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.reader = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.reader.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- helpers
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_traffic():
    """dram bytes per launch of the forward kernel from the committed ncu
    --set full summary (profiles/ncu_fwd_summary.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_fwd_summary.json")
    try:
        with open(path) as f:
            doc = json.load(f)
        return doc.get("dram_bytes_per_launch"), doc.get("workload")
    except (OSError, ValueError):
        return None, None


def cpu_baseline_sample(n, heads, batch, tiles, workers):
    """Reference CPU algorithm (oracle/scan_port.py = engine.scan_forward) on
    `tiles` whole 64-query tiles of the workload; returns (TFLOP/s, seconds,
    description)."""
    import oracle

    Q, K, V = oracle.generate(0, "regular", b=batch, h=heads, n=n, d=64, d_v=64,
                              dtype=np.float32)
    rng = np.random.default_rng(0)
    starts = [(0, int(rng.integers(0, heads)), 64 * int(rng.integers(0, n // 64)))
              for _ in range(tiles)]
    t0 = time.perf_counter()
    oracle.scan_forward_port(Q, K, V, block_size=128, tile_q=64, workers=workers, tiles=starts)
    dt = time.perf_counter() - t0
    fl = tiles * flops(1, 1, 64, n)
    desc = (f"{tiles} x 64-query tiles of B{batch} H{heads} n{n} d64 (reference blocked scan, "
            f"B=128, tile_q=64, {workers} threads), extrapolated linearly in tiles")
    return fl / dt / 1e12, dt, desc


def cpu_full_configs(workers):
    """the reference CPU algorithm timed in full on the small
    BASELINE configs (C1, C2 and C3 at n = 1K), on the same host threads."""
    import oracle

    rows = []
    for name, (B, H, n) in (("C1", (1, 1, 1024)), ("C2 BERT-base", (8, 12, 512)),
                            ("C3 n=1K", (1, 16, 1024))):
        Q, K, V = oracle.generate(0, "regular", b=B, h=H, n=n, d=64, d_v=64, dtype=np.float32)
        t0 = time.perf_counter()
        oracle.scan_forward_port(Q, K, V, block_size=128, tile_q=64, workers=workers)
        dt = time.perf_counter() - t0
        rows.append({"config": name, "B": B, "H": H, "n": n, "seconds": dt,
                     "tflops": flops(B, H, n, n) / dt / 1e12, "cores": workers,
                     "kind": "port", "timed": "full problem"})
    return rows


def _cpu_workers(args):
    cores = os.cpu_count() or 1
    # each worker holds ~0.8 GB of (T, n, d_v) scan lanes at n = 16K; bound RAM
    return args.cpu_workers or max(1, min(cores, 16))


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    workers = _cpu_workers(args)
    tiles = args.cpu_sample_tiles or workers
    n, H, B = args.n, args.heads, args.batch
    for _ in range(args.warmup):
        cpu_baseline_sample(min(n, 2048), 1, 1, 1, 1)
    vals, secs = [], []
    desc = ""
    for _ in range(args.steps):
        v, dt, desc = cpu_baseline_sample(n, H, B, tiles, workers)
        vals.append(v)
        secs.append(dt)
    value = float(np.median(vals))
    full_ms = flops(B, H, n, n) / (value * 1e12) * 1e3
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": full_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (scanattn regular generator, seed 0)",
        "config": {"workload": f"C3 FP32 attention B{B} H{H} n{n} d64 (bounded CPU sample)",
                   "B": B, "H": H, "n": n, "d": 64, "dv": 64},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": workers, "kind": "port",
                         "sample": desc, "sample_seconds_median": float(np.median(secs))},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2604_23798_b200 as elsa
    from paper_2604_23798_b200 import dist as edist

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.dist_path:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=dev)
    sharded = world > 1 or args.dist_path
    B, H, n = args.batch, args.heads, args.n
    fl = flops(B, H, n, n)
    stream = torch.cuda.current_stream(dev)

    # ---- inputs (same generator as the reference, tensorio.py:177-195) ----
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    q = torch.randn(B, H, n, 64, device=dev, generator=gen)
    k = torch.randn(B, H, n, 64, device=dev, generator=gen)
    v = torch.randn(B, H, n, 64, device=dev, generator=gen)
    chunks = 8 if world <= 8 and 8 % world == 0 else world
    if sharded:
        k_loc, v_loc, off = edist.shard_kv(k, v, rank, world, chunks)
        k_loc, v_loc = k_loc.contiguous(), v_loc.contiguous()

    launches = [0]
    exchange = [args.exchange]

    def step():
        if not sharded:
            y = elsa.scaled_dot_product_attention(q, k, v)
            launches[0] += elsa.last_launch_count()
            return y
        if args.shard == "q":
            r = edist.query_sharded_attention(q, k, v)
        else:
            r = edist.kv_sharded_attention(q, k_loc, v_loc, off, n, chunks=chunks, gather=False,
                                           exchange=exchange[0])
        launches[0] += 2 * (chunks // world) + 1
        return r

    if sharded and args.shard == "kv" and exchange[0] == "peer":
        # the symmetric-memory rendezvous needs peer access between every pair
        # of GPUs; if this node cannot provide it, measure the NCCL exchange
        try:
            step()
            torch.cuda.synchronize()
            ok = torch.ones(1, device=dev)
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] peer exchange unavailable ({str(exc)[:120]}); using NCCL",
                  file=sys.stderr)
            ok = torch.zeros(1, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() < 1:
            exchange[0] = "nccl"

    def barrier():
        if sharded:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    launches[0] = 0
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_total = e0.elapsed_time(e1)
    clock_info = clocks.stop()
    timed_launches = launches[0]
    if sharded:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms = ms_total / args.steps
    value = fl / (ms * 1e-3) / 1e12

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e and sharded:
        # each rank: H2D of Q and its K/V shard, the KV-sharded forward, D2H of
        # its Y row slice (the ranks' slices together are the whole Y)
        k_src, v_src = (k, v) if args.shard == "q" else (k_loc, v_loc)
        hq = q.cpu().pin_memory()
        hk, hv = k_src.cpu().pin_memory(), v_src.cpu().pin_memory()
        dq, dk, dv_ = torch.empty_like(q), torch.empty_like(k_src), torch.empty_like(v_src)
        hy = [None]

        def e2e_step_dist():
            dq.copy_(hq, non_blocking=True)
            dk.copy_(hk, non_blocking=True)
            dv_.copy_(hv, non_blocking=True)
            if args.shard == "q":
                _, yr = edist.query_sharded_attention(dq, dk, dv_)
            else:
                _, yr = edist.kv_sharded_attention(dq, dk, dv_, off, n, chunks=chunks,
                                                   gather=False, exchange=exchange[0])
            if hy[0] is None:
                hy[0] = torch.empty(yr.shape, dtype=yr.dtype).pin_memory()
            hy[0].copy_(yr, non_blocking=True)

        for _ in range(2):
            e2e_step_dist()
        torch.cuda.synchronize()
        barrier()
        steps_e2e = max(3, min(args.steps, 10))
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(steps_e2e):
            e2e_step_dist()
        a1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a0.elapsed_time(a1) / steps_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        e2e = {"value": fl / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": (q.numel() + k_src.numel() + v_src.numel()) * 4 * world,
               "d2h_bytes_per_step": hy[0].numel() * 4 * world, "steps": steps_e2e,
               "api": "paper_2604_23798_b200.dist.kv_sharded_attention per rank, pinned host "
                      "buffers (bytes summed over ranks; max-over-ranks time)"}
    if not args.no_e2e and not sharded:
        hq = q.cpu().pin_memory()
        hk = k.cpu().pin_memory()
        hv = v.cpu().pin_memory()
        hy = torch.empty((B, H, n, 64), dtype=torch.float32).pin_memory()

        def e2e_step():
            # the public host-buffer entry point (elsa_fwd_f32_host): per-head-group
            # H2D -> forward -> D2H pipelined on internal streams; the current
            # stream waits for the last D2H
            elsa.attention_from_host(hq, hk, hv, out=hy, sync=False)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        steps_e2e = max(3, min(args.steps, 10))
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(steps_e2e):
            e2e_step()
        a1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a0.elapsed_time(a1) / steps_e2e
        e2e = {"value": fl / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 3 * q.numel() * 4, "d2h_bytes_per_step": hy.numel() * 4,
               "steps": steps_e2e,
               "api": "paper_2604_23798_b200.attention_from_host -> elsa_fwd_f32_host (C-ABI), "
                      "pinned host buffers"}

    # ---- roofline: FFMA peak (spec clock) and the K4 microbenchmark ----
    peaks = measured_peaks()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    spec_peak = SMS * FFMA_LANES * 2 * fmax * 1e6 / 1e12
    k4 = None
    try:
        k4 = elsa.ffma_peak_tflops(dev)
    except Exception:  # noqa: BLE001
        k4 = None
    traffic, traffic_workload = ncu_traffic()
    roofline = {
        "bound": "ffma", "achieved": value, "peak": spec_peak, "unit": "TFLOP/s",
        "frac": value / spec_peak,
        "peak_source": f"148 SM x 128 FP32 lanes x 2 x {fmax:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
        "k4_ffma_measured": k4, "frac_of_k4": (value / k4) if k4 else None,
        "traffic": traffic, "traffic_workload": traffic_workload,
        "algorithmic_bytes_per_launch": 4 * B * H * (n * 64 * 3 + n * 64),
        "kernel": "elsa::fwd_f32_kernel (" + elsa.describe_plan(q, k, v) + ")" if not sharded else "elsa::fwd_f32_kernel",
        "measurement": "CUDA events on the launching stream around the K timed steps; "
                       "one kernel launch per step at this shape",
    }

    # ---- sweep (kernel-only: CUDA-graph replays, L2 flushed between them) ----
    sweep = []
    if not args.no_sweep and not sharded:
        flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
        cases = [(1, 16, nn) for nn in (1024, 2048, 4096, 8192, 16384)] + [(8, 12, 512), (1, 1, 1024)]
        for (bb, hh, nn) in cases:
            qq = torch.randn(bb, hh, nn, 64, device=dev)
            kk = torch.randn(bb, hh, nn, 64, device=dev)
            vv = torch.randn(bb, hh, nn, 64, device=dev)
            for _ in range(3):
                elsa.scaled_dot_product_attention(qq, kk, vv)
            torch.cuda.synchronize()
            # capture one call so host-side Python overhead stays out of the
            # measurement; replays are enqueued back to back (no host idle gaps)
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(dev)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(graph, stream=cap):
                    elsa.scaled_dot_product_attention(qq, kk, vv)
            torch.cuda.synchronize()
            reps = 30 if nn <= 4096 else 8
            evs = []
            for _ in range(reps):
                flush.fill_(1.0)
                s0 = torch.cuda.Event(enable_timing=True)
                s1 = torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                graph.replay()
                s1.record(stream)
                evs.append((s0, s1))
            torch.cuda.synchronize()
            times = [a.elapsed_time(b) for a, b in evs[2:]]
            t_ms = float(np.median(times))
            tf = flops(bb, hh, nn, nn) / (t_ms * 1e-3) / 1e12
            sweep.append({"B": bb, "H": hh, "n": nn, "ms": t_ms, "tflops": tf,
                          "frac_ffma_peak": tf / spec_peak,
                          "plan": elsa.describe_plan(qq, kk, vv)})
            del qq, kk, vv, graph
        # GPU comparator on the same box: torch SDPA FP32 (TF32 off), the paper's ME-SDPA
        try:
            torch.backends.cuda.matmul.allow_tf32 = False
            torch.backends.cudnn.allow_tf32 = False
            for _ in range(2):
                torch.nn.functional.scaled_dot_product_attention(q, k, v)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(3):
                torch.nn.functional.scaled_dot_product_attention(q, k, v)
            s1.record(stream)
            torch.cuda.synchronize()
            tms = s0.elapsed_time(s1) / 3
            sweep.append({"comparator": "torch.nn.functional.scaled_dot_product_attention fp32",
                          "B": B, "H": H, "n": n, "ms": tms, "tflops": fl / (tms * 1e-3) / 1e12})
        except Exception as exc:  # noqa: BLE001
            sweep.append({"comparator": "torch sdpa fp32", "error": str(exc)[:200]})
        # the FP16/BF16 variant (K5, tcgen05) on the same problem, for comparison
        # (BASELINE configs[4]); flops 4*B*H*n^2*64, same as the FP32 count
        for dt, nm, dh in ((torch.bfloat16, "bf16", 64), (torch.float16, "fp16", 64),
                           (torch.bfloat16, "bf16", 128)):
            try:
                if dh == 64:
                    q16, k16, v16 = q.to(dt), k.to(dt), v.to(dt)
                else:  # wider heads (d = dv = 128), same sequence shape
                    q16, k16, v16 = (torch.randn(B, H, n, dh, device=dev, generator=gen).to(dt)
                                     for _ in range(3))
                fl16 = 4.0 * B * H * n * n * dh
                row = {"variant": f"elsa {nm} (tcgen05)", "B": B, "H": H, "n": n, "d": dh}
                for label, fn in (("elsa", lambda: elsa.scaled_dot_product_attention(q16, k16, v16)),
                                  ("torch", lambda: torch.nn.functional.scaled_dot_product_attention(
                                      q16, k16, v16))):
                    for _ in range(2):
                        fn()
                    s0 = torch.cuda.Event(enable_timing=True)
                    s1 = torch.cuda.Event(enable_timing=True)
                    s0.record(stream)
                    for _ in range(5):
                        fn()
                    s1.record(stream)
                    torch.cuda.synchronize()
                    tms = s0.elapsed_time(s1) / 5
                    row[f"{label}_ms"] = tms
                    row[f"{label}_tflops"] = fl16 / (tms * 1e-3) / 1e12
                sweep.append(row)
                del q16, k16, v16
            except Exception as exc:  # noqa: BLE001
                sweep.append({"variant": f"elsa {nm}", "error": str(exc)[:200]})

    # ---- CPU baseline: the reference's algorithm on the host cores (rank 0, N=1) ----
    cpu = None
    if rank == 0 and not sharded and not args.no_cpu_baseline:
        workers = _cpu_workers(args)
        tiles = args.cpu_sample_tiles or workers
        val, secs, desc = cpu_baseline_sample(n, H, B, tiles, workers)
        cpu = {"value": val, "unit": "TFLOP/s", "cores": workers, "kind": "port",
               "sample": desc, "seconds": secs,
               "full_small_configs": cpu_full_configs(workers)}

    if sharded and args.shard == "kv":
        # per-rank working set of one step: all of Q, this rank's K/V shard and
        # its chunk states (m, S, W for every query row)
        per = chunks // world
        ws_mb = (q.numel() + k_loc.numel() + v_loc.numel()
                 + per * B * H * n * (2 + 64)) * 4 / 1e6
        l2_note = ("per-rank step working set %.0f MB (Q, K/V shard, chunk states) > 126 MB L2; "
                   "sweep flushes L2 (256 MB write) between timed iterations" % ws_mb)
    else:
        l2_note = ("inputs 3x%.0f MB > 126 MB L2; sweep flushes L2 (256 MB write) "
                   "between timed iterations" % (q.numel() * 4 / 1e6))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic N(0,1) Q/K/V (torch.randn), resident in HBM",
            "config": {"workload": f"C3 FP32 attention B{B} H{H} n{n} d64 dv64"
                                   + (f", KV-sharded over {world} GPUs ({chunks} chunks)"
                                      if sharded else ""),
                       "B": B, "H": H, "n": n, "d": 64, "dv": 64,
                       "l2": l2_note,
                       "parallelism": f"kv-shard{world}" if sharded else "single GPU",
                       "exchange": (exchange[0] if args.shard == "kv" else "none (query-sharded)")
                                   if sharded else None},
            "e2e": e2e, "gpu_launches": timed_launches, "clocks": clock_info,
            "roofline": roofline, "cpu_baseline": cpu, "sweep": sweep,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
