#!/usr/bin/env python
"""ELSA FP32 exact attention on B200 — the driver's benchmark.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl elsa|reference]

Headline workload (BASELINE.json configs[2], the config its metric is quoted
on): FP32 attention B=1 H=16 d=dv=64 at n=16384 per GPU — one "step" is one
full forward over the (B, H, n, d) problem. `value` is whole-job TFLOP/s with
algorithmic flops 2*B*H*n^2*(d+dv) (QK^T + PV, FMA = 2; exps not counted),
inputs resident in HBM (3 x 67 MB > the 126 MB L2, so consecutive steps do not
hit in L2). `e2e` is the same metric through the public host-buffer entry
point (`paper_2604_23798_b200.attention_from_host` -> C-ABI
`elsa_fwd_f32_host`) with pinned host buffers: H2D of Q/K/V and D2H of Y
inside the timed region, pipelined per head group under the kernels.
`parity` checks sampled rows of the Y the timed steps produced against FP64.

N > 1 (torchrun, one rank per GPU, NCCL): the work shards over batch x heads
(BASELINE north_star) — the global problem is B=N (one C3-16K problem per
GPU), split into contiguous (b, h, q) row slices by
`dist.query_sharded_attention`, no data-path collective (`scaling: weak`).
`strong` times the fixed B=1 problem over the same row slicing.

`long_context` (every N): C4 (B1 H16 n=65536) and C5 (B1 H8 n=2^20) — at
N = 1 the single-GPU forward, at N > 1 KV-sharded over the ranks
(Proposition 1: per-chunk (m, S, W) states, fused
peer-memory merge over NVLink), strong scaling of a fixed problem, each with
FP64 sampled-row parity.

The sweep (N = 1: 1K..16K, BERT-base, the single-head config, the FP32 SDPA
comparator and the 16-bit tcgen05 variant) flushes the L2 between timed
iterations.

`--impl reference` times the reference's own CPU algorithm (the blocked
scan of scanattn.engine.scan_forward, restated bit-exactly in
oracle/scan_port.py) on the host cores, on a bounded sample of the same
workload (whole 64-query tiles), and reports the same metric.
"""

from __future__ import annotations

import argparse
import datetime
import glob
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
U32 = 2.0 ** -24


def flops(b, h, n_q, n_kv, d=64, dv=64):
    return 2.0 * b * h * n_q * n_kv * (d + dv)


def scan_depth(n, block=128):
    """L(n, B) of engine.py:47-55 (the parity bound's depth factor)."""
    def clog2(x):
        return 0 if x <= 1 else (int(x) - 1).bit_length()
    return clog2(min(block, n)) + 2 * clog2(-(-n // block)) + 3


def bound(n):
    return U32 * scan_depth(n) * 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["elsa", "reference"], default="elsa")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=1, help="batch per GPU")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--sampled-parity", action="store_true",
                    help="N = 1: check 64 sampled rows instead of every row of the timed output")
    ap.add_argument("--long", default="c4,c5",
                    help="long-context configs to time at every N (comma list of c4, c5; "
                         "'none' to skip)")
    ap.add_argument("--cpu-sample-tiles", type=int, default=0,
                    help="64-query tiles per CPU sample (0 = one per worker)")
    ap.add_argument("--cpu-workers", type=int, default=0)
    ap.add_argument("--dist-path", action="store_true",
                    help="run the N > 1 code paths even at N = 1 (a world-size-1 NCCL group)")
    ap.add_argument("--shard", choices=["q", "kv"], default="q",
                    help="headline at N > 1: batch x heads row slices (no exchange, the "
                         "natural sharding) or KV-sharded (Proposition 1)")
    ap.add_argument("--exchange", choices=["auto", "peer", "nccl"], default="auto",
                    help="KV-sharded runs: fused symmetric-memory peer merge or NCCL "
                         "all_to_all + merge kernel (auto = peer on NCCL groups)")
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

    def wait_first(self, timeout):
        """Block until the sampler produced two samples (NVML initialised and
        polling), then drop them: only samples of the timed region count."""
        t0 = time.time()
        while self.proc is not None and len(self.lines) < 2 and time.time() - t0 < timeout:
            time.sleep(0.02)
        time.sleep(0.1)
        del self.lines[:]

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


def host_info():
    """The host the CPU baseline runs on (engine.py:88-89: the reference's
    default is workers='auto' -> os.cpu_count())."""
    cores = os.cpu_count() or 1
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = cores
    try:
        import psutil
        mem_gb = psutil.virtual_memory().available / 1e9
    except Exception:  # noqa: BLE001
        mem_gb = None
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cores": cores, "usable_cores": usable, "cpu_model": model,
            "mem_available_gb": mem_gb}


def _cpu_workers(args, gb_per_worker=0.0):
    """All usable host cores (the reference's workers='auto'), bounded only by
    RAM when each worker holds `gb_per_worker` of scan lanes."""
    if args.cpu_workers:
        return args.cpu_workers
    info = host_info()
    w = info["usable_cores"]
    if gb_per_worker and info["mem_available_gb"]:
        w = min(w, max(1, int(0.6 * info["mem_available_gb"] / gb_per_worker)))
    return max(1, w)


# the reference's scan of one 64-query tile holds ~0.8 GB of (T, n, d_v) lanes at n = 16K
def _lane_gb(n):
    return 0.8 * n / 16384


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
    BASELINE configs (C1, C2 and C3 at n = 1K and 2K), on all host threads."""
    import oracle

    rows = []
    for name, (B, H, n) in (("C1", (1, 1, 1024)), ("C2 BERT-base", (8, 12, 512)),
                            ("C3 n=1K", (1, 16, 1024)), ("C3 n=2K", (1, 16, 2048))):
        Q, K, V = oracle.generate(0, "regular", b=B, h=H, n=n, d=64, d_v=64, dtype=np.float32)
        t0 = time.perf_counter()
        oracle.scan_forward_port(Q, K, V, block_size=128, tile_q=64, workers=workers)
        dt = time.perf_counter() - t0
        rows.append({"config": name, "B": B, "H": H, "n": n, "seconds": dt,
                     "tflops": flops(B, H, n, n) / dt / 1e12, "cores": workers,
                     "kind": "port", "timed": "full problem"})
    return rows


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n, H, B = args.n, args.heads, args.batch
    workers = _cpu_workers(args, _lane_gb(n))
    tiles = args.cpu_sample_tiles or workers
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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (scanattn regular generator, seed 0)",
        "config": {"workload": f"C3 FP32 attention B{B} H{H} n{n} d64 (bounded CPU sample)",
                   "B": B, "H": H, "n": n, "d": 64, "dv": 64},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": workers, "kind": "port",
                         "sample": desc, "sample_seconds_median": float(np.median(secs)),
                         **host_info()},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
class Ctx:
    """Rank / device / process-group plumbing shared by the timed sections."""

    def __init__(self, args):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        if self.world > 1 or args.dist_path:
            # NCCL's communicator-init lines (ranks, NVLink/NVLS topology) go to a
            # per-rank file (set before NCCL is loaded) and are echoed to stderr:
            # the evidence that N ranks formed one communicator (stdout stays
            # one JSON line)
            if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
                os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ["NCCL_DEBUG_FILE"] = f"/tmp/elsa_nccl.{os.getpid()}.log"
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.distributed = self.world > 1 or args.dist_path
        self.comm = None
        if self.distributed:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", str(self.world))
            # a failed rank must not park the others for NCCL's default 10
            # minutes: the longest gap between collectives here is one C5
            # KV-sharded step (~20 s at N = 2)
            dist.init_process_group("nccl", device_id=self.dev,
                                    timeout=datetime.timedelta(minutes=5))
            t = torch.ones(1, device=self.dev)
            dist.all_reduce(t)
            torch.cuda.synchronize()
            self.comm = self._nccl_lines(int(t.item()))
        self.stream = torch.cuda.current_stream(self.dev)

    def _nccl_lines(self, nranks_seen):
        lines = []
        for path in glob.glob(f"/tmp/elsa_nccl.{os.getpid()}.log*"):
            try:
                with open(path) as f:
                    lines += [ln.rstrip() for ln in f]
            except OSError:
                pass
        for ln in lines:
            if "Init COMPLETE" in ln or "comm 0x" in ln or "NVLS" in ln or "P2P" in ln:
                print(f"[rank {self.rank}] {ln}", file=sys.stderr)
        version = next((ln.split("NCCL version", 1)[1].strip().split()[0]
                        for ln in lines if "NCCL version" in ln), None)
        complete = [ln for ln in lines if "Init COMPLETE" in ln]
        nvls = any("NVLS" in ln and "enabled" in ln.lower() for ln in lines)
        return {"backend": "nccl", "world": self.world, "all_reduce_ranks": nranks_seen,
                "nccl_version": version, "init_complete_lines": len(complete),
                "init_line": complete[0][-200:] if complete else None, "nvls_logged": nvls}

    def barrier(self):
        if self.distributed:
            self.dist.barrier()

    def max_over_ranks(self, x):
        if not self.distributed:
            return x
        t = self.torch.tensor([float(x)], device=self.dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x):
        if not self.distributed:
            return x
        t = self.torch.tensor([float(x)], device=self.dev, dtype=self.torch.float64)
        self.dist.all_reduce(t)
        return float(t.item())

    def timed(self, fn, steps):
        """max-over-ranks ms per call of `fn` over `steps` calls: barrier +
        synchronize on both sides, CUDA events on the launching stream."""
        torch = self.torch
        self.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        out = None
        for _ in range(steps):
            out = fn()
        e1.record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        return self.max_over_ranks(e0.elapsed_time(e1) / steps), out


def sampled_parity(q, k, v, y_rows, row_lo, rows_wanted, seed):
    """FP64 check of sampled output rows (oracles.py:92-98 restated in numpy:
    row-max-stabilised softmax in float64). `y_rows` holds the flattened
    (b, h, q) rows [row_lo, row_lo + len); returns the max per-row relative L2
    error (verify.py:336-338) and the rows checked."""
    import torch
    B, H, n_q, d = q.shape
    n_kv = k.shape[2]
    total = y_rows.shape[0]
    rng = np.random.default_rng(seed)
    picks = sorted(set([0, total - 1] + rng.integers(0, total, max(rows_wanted - 2, 0)).tolist()))
    by_head = {}
    for p in picks:
        bh, r = divmod(row_lo + p, n_q)
        by_head.setdefault(bh, []).append((p, r))
    sc = 1.0 / math.sqrt(d)
    errs = []
    for bh, items in by_head.items():
        b, h = divmod(bh, H)
        K = k[b, h].to(torch.float64).cpu().numpy()
        V = v[b, h].to(torch.float64).cpu().numpy()
        qs = q[b, h, [r for _, r in items]].to(torch.float64).cpu().numpy()
        got = y_rows[[p for p, _ in items]].to(torch.float64).cpu().numpy()
        s = (qs @ K.T) * sc
        s -= s.max(axis=1, keepdims=True)
        np.exp(s, out=s)
        ref = (s @ V) / s.sum(axis=1, keepdims=True)
        errs += list(np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1))
        del K, V, s
    return (max(errs) if errs else 0.0), len(errs)


def full_parity(q, k, v, y_rows):
    """Every output row against the FP64 oracle (oracles.py:92-98 restated in
    numpy float64, query rows in chunks); max per-row relative L2 error
    (verify.py:336-338) and the row count."""
    import torch
    f64 = torch.float64
    B, H, n_q, d = q.shape
    sc = 1.0 / math.sqrt(d)
    Y = y_rows.reshape(B, H, n_q, -1)
    worst, rows = 0.0, 0
    for b in range(B):
        for h in range(H):
            K = k[b, h].to(f64).cpu().numpy()
            V = v[b, h].to(f64).cpu().numpy()
            Qh = q[b, h].to(f64).cpu().numpy()
            Yh = Y[b, h].to(f64).cpu().numpy()
            for r0 in range(0, n_q, 2048):
                s = (Qh[r0:r0 + 2048] @ K.T) * sc
                s -= s.max(axis=1, keepdims=True)
                np.exp(s, out=s)
                ref = (s @ V) / s.sum(axis=1, keepdims=True)
                e = np.linalg.norm(Yh[r0:r0 + 2048] - ref, axis=1) / np.linalg.norm(ref, axis=1)
                worst = max(worst, float(e.max()))
                rows += e.size
            del K, V, Qh, Yh
    return worst, rows


def _parity_block(ctx, err, rows, n_kv):
    err = ctx.max_over_ranks(err)
    rows = int(ctx.sum_over_ranks(rows))
    thr = bound(n_kv)
    return {"max_err": err, "bound": thr, "rows": rows, "pass": bool(err <= thr),
            "oracle": "FP64 row-max-stabilised softmax on the host (oracles.py:92-98), "
                      "per-row relative L2 (verify.py:336-338), bound u*L(n,128)*8 "
                      "(verify.py:339-343)"}


def headline(args, ctx, elsa, edist):
    """The C3-16K step: N = 1 the single-GPU forward, N > 1 the B = N global
    problem over (b, h, q) row slices (or KV-sharded with --shard kv)."""
    torch = ctx.torch
    world, rank, dev = ctx.world, ctx.rank, ctx.dev
    H, n = args.heads, args.n
    Bg = args.batch * world if ctx.distributed and args.shard == "q" else args.batch
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    q = torch.randn(Bg, H, n, 64, device=dev, generator=gen)
    k = torch.randn(Bg, H, n, 64, device=dev, generator=gen)
    v = torch.randn(Bg, H, n, 64, device=dev, generator=gen)
    launches = [0]
    chunks = edist.DEFAULT_CHUNKS if world <= 8 and 8 % world == 0 else world
    state = {}

    if not ctx.distributed:
        def step():
            y = elsa.scaled_dot_product_attention(q, k, v)
            launches[0] += elsa.last_launch_count()
            return 0, y.reshape(-1, 64)
    elif args.shard == "q":
        def step():
            lo, y = edist.query_sharded_attention(q, k, v)
            launches[0] += edist.last_launch_count()
            return lo, y
    else:
        k_loc, v_loc, off = edist.shard_kv(k, v, rank, world, chunks)
        k_loc, v_loc = k_loc.contiguous(), v_loc.contiguous()
        state["kv"] = (k_loc, v_loc, off)

        def step():
            r = edist.kv_sharded_attention(q, k_loc, v_loc, off, n, chunks=chunks, gather=False,
                                           exchange=args.exchange)
            launches[0] += edist.last_launch_count()
            return r

    warm = max(args.warmup, 3)
    # the sampler starts before the warm-up: on a fresh box nvidia-smi's first
    # NVML initialisation stalls the GPU for milliseconds (measured: the first
    # bench run on a box 22.8 ms/step, the next ones 19.18), so it must be
    # sampling steadily before the timed region opens
    clocks = ClockSampler(ctx.local)
    clocks.start()
    # at least W steps and at least ~0.5 s of GPU work, so the SM clocks have
    # left the idle state before timing (the reported warmup is the count run)
    t_warm = time.time()
    done = 0
    # (N > 1: a fixed count, the KV-sharded steps hold collectives)
    while done < warm or (not ctx.distributed and time.time() - t_warm < 0.5):
        step()
        done += 1
        if done >= warm:
            torch.cuda.synchronize()
    warm = done
    clocks.wait_first(timeout=10.0)
    launches[0] = 0
    ms, (lo, y_rows) = ctx.timed(step, args.steps)
    clock_info = clocks.stop()
    timed_launches = launches[0]
    fl = flops(Bg, H, n, n)
    value = fl / (ms * 1e-3) / 1e12
    parity = None
    if not args.no_parity:
        if world == 1 and not args.sampled_parity:
            # every row of the timed output against the FP64 oracle (~20 s of
            # host BLAS at 16K)
            err, cnt = full_parity(q, k, v, y_rows)
            parity = _parity_block(ctx, err, cnt, n)
            parity["rows_checked"] = "all"
        else:
            err, cnt = sampled_parity(q, k, v, y_rows, lo, max(8, 64 // world), seed=rank + 1)
            parity = _parity_block(ctx, err, cnt, n)
    plan = elsa.describe_plan(q[:1], k[:1], v[:1])
    return dict(q=q, k=k, v=v, Bg=Bg, fl=fl, ms=ms, value=value, clocks=clock_info,
                launches=timed_launches, parity=parity, plan=plan, chunks=chunks,
                warmup=warm, state=state)


def strong_c3(args, ctx, elsa, edist, hl):
    """N > 1: the fixed B1 H16 n16K problem over the ranks' row slices."""
    q, k, v = (t[:1] for t in (hl["q"], hl["k"], hl["v"]))
    for _ in range(2):
        edist.query_sharded_attention(q, k, v)
    ms, _ = ctx.timed(lambda: edist.query_sharded_attention(q, k, v), max(3, args.steps // 2))
    fl = flops(1, args.heads, args.n, args.n)
    return {"workload": f"C3 B1 H{args.heads} n{args.n} d64 (fixed), (b, h, q) row slices over "
                        f"{ctx.world} GPUs", "ms_per_step": ms,
            "value": fl / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "scaling": "strong"}


def e2e_block(args, ctx, elsa, hl):
    """Each rank: its rows' Q/K/V from pinned host memory -> GPU -> Y rows back
    to pinned host memory, through attention_from_host (C-ABI
    elsa_fwd_f32_host, pipelined per head group); N > 1: the rank's own batch
    elements (its row slice of the B = N problem)."""
    torch = ctx.torch
    q, k, v = hl["q"], hl["k"], hl["v"]
    if ctx.distributed and args.shard == "q":
        b0 = ctx.rank * args.batch
        q, k, v = (t[b0:b0 + args.batch] for t in (q, k, v))
    elif ctx.distributed:
        return None  # the KV-sharded headline has no host-buffer entry
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hy = torch.empty(tuple(q.shape[:-1]) + (64,), dtype=torch.float32).pin_memory()

    def e2e_step():
        elsa.attention_from_host(hq, hk, hv, out=hy, sync=False)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    steps_e2e = max(3, min(args.steps, 10))
    ms, _ = ctx.timed(e2e_step, steps_e2e)
    fl = hl["fl"]
    h2d = ctx.sum_over_ranks((hq.numel() + hk.numel() + hv.numel()) * 4)
    d2h = ctx.sum_over_ranks(hy.numel() * 4)
    return {"value": fl / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps_e2e,
            "api": "paper_2604_23798_b200.attention_from_host -> elsa_fwd_f32_host (C-ABI), "
                   "pinned host buffers" + (", each rank its own batch elements (bytes summed "
                                            "over ranks, max-over-ranks time)"
                                            if ctx.distributed else "")}


LONG = {"c4": ("C4", 1, 16, 65536), "c5": ("C5", 1, 8, 1 << 20)}


def probe_exchange(args, ctx, edist):
    """The KV-sharded exchange this node supports: the fused peer merge needs
    symmetric (peer-mapped) memory between every pair of GPUs; a tiny
    sharded problem is run with it on every rank and the ranks agree (MIN)
    whether it worked, else the NCCL all_to_all exchange is used."""
    torch = ctx.torch
    want = edist.resolve_exchange(args.exchange, torch.empty(0, device=ctx.dev))
    if not ctx.distributed or want != "peer":
        return want, None
    chunks = edist.DEFAULT_CHUNKS if ctx.world <= 8 and 8 % ctx.world == 0 else ctx.world
    err = None
    try:
        g = torch.Generator(device=ctx.dev)
        g.manual_seed(3)
        q, k, v = (torch.randn(1, 2, 512, 64, device=ctx.dev, generator=g) for _ in range(3))
        kl, vl, off = edist.shard_kv(k, v, ctx.rank, ctx.world, chunks)
        edist.kv_sharded_attention(q, kl.contiguous(), vl.contiguous(), off, 512, chunks=chunks,
                                   gather=False, exchange="peer")
        torch.cuda.synchronize()
        ok = torch.ones(1, device=ctx.dev)
    except Exception as exc:  # noqa: BLE001
        err = f"{type(exc).__name__}: {str(exc)[:160]}"
        print(f"[bench rank {ctx.rank}] peer exchange unavailable ({err}); using NCCL",
              file=sys.stderr)
        ok = torch.zeros(1, device=ctx.dev)
    ctx.dist.all_reduce(ok, op=ctx.dist.ReduceOp.MIN)
    edist.release_peer_buffers()
    return ("peer" if ok.item() > 0 else "nccl"), err


def long_context(args, ctx, elsa, edist, spec_peak):
    """C4 / C5 at this N: the single-GPU forward at N = 1, KV-sharded over the
    ranks at N > 1 (strong scaling of the fixed problem)."""
    torch = ctx.torch
    out = []
    names = [x.strip() for x in args.long.split(",") if x.strip() and x.strip() != "none"]
    exchange, probe_err = probe_exchange(args, ctx, edist) if names else (None, None)
    for key in names:
        try:
            out.append(_long_one(args, ctx, elsa, edist, spec_peak, key, exchange, probe_err))
        except Exception as exc:  # noqa: BLE001 - keep the headline line alive
            print(f"[bench rank {ctx.rank}] long-context {key} failed: {exc}", file=sys.stderr)
            out.append({"config": LONG[key][0], "error": f"{type(exc).__name__}: {str(exc)[:200]}"})
            torch.cuda.empty_cache()
    return out


def _long_one(args, ctx, elsa, edist, spec_peak, key, exchange, probe_err):
    torch = ctx.torch
    tag, B, H, n = LONG[key]
    gen = torch.Generator(device=ctx.dev)
    gen.manual_seed(64 + n % 977)
    q = torch.randn(B, H, n, 64, device=ctx.dev, generator=gen)
    k = torch.randn(B, H, n, 64, device=ctx.dev, generator=gen)
    v = torch.randn(B, H, n, 64, device=ctx.dev, generator=gen)
    fl = flops(B, H, n, n)
    steps = 3 if key == "c4" else 1
    launches = [0]
    row = {"config": tag, "workload": f"{tag} FP32 attention B{B} H{H} n{n} d64 dv64",
           "n_gpus": ctx.world, "scaling": "strong"}
    if not ctx.distributed:
        def step():
            y = elsa.scaled_dot_product_attention(q, k, v)
            launches[0] += elsa.last_launch_count()
            return 0, y.reshape(-1, 64)
        # C5 at N = 1 is a ~39 s step: warm it on the first 8192 query rows
        # (same keys, same kernel); C4 warms on the full problem
        if key == "c5":
            elsa.scaled_dot_product_attention(q[:, :, :8192], k, v)
        else:
            step()
        row["path"] = "single GPU: elsa_fwd_f32 (" + elsa.describe_plan(q, k, v) + ")"
    else:
        chunks = edist.DEFAULT_CHUNKS if ctx.world <= 8 and 8 % ctx.world == 0 else ctx.world
        kl, vl, off = edist.shard_kv(k, v, ctx.rank, ctx.world, chunks)
        kl, vl = kl.contiguous(), vl.contiguous()
        ex = [exchange]

        def step():
            r = edist.kv_sharded_attention(q, kl, vl, off, n, chunks=chunks, gather=False,
                                           exchange=ex[0])
            launches[0] += edist.last_launch_count()
            return r
        step()  # full warm-up: rendezvous of the peer buffer, workspaces
        row["path"] = (f"KV-sharded: {chunks} global key chunks, {chunks // ctx.world} per "
                       f"rank, exchange={exchange}"
                       + (f" (peer probe failed: {probe_err})" if probe_err else ""))
        row["per_rank_keys"] = int(kl.shape[2])
    torch.cuda.synchronize()
    launches[0] = 0
    ms, (lo, y_rows) = ctx.timed(step, steps)
    tf = fl / (ms * 1e-3) / 1e12
    row.update({"steps": steps, "ms_per_step": ms, "value": tf, "unit": "TFLOP/s",
                "gpu_launches_per_step": ctx.max_over_ranks(launches[0]) / steps,
                "frac_ffma_peak_per_gpu": tf / (ctx.world * spec_peak)})
    if not args.no_parity:
        err, cnt = sampled_parity(q, k, v, y_rows, lo, 8 if key == "c5" else 16,
                                  seed=100 + ctx.rank)
        row["parity"] = _parity_block(ctx, err, cnt, n)
    del q, k, v, y_rows
    if ctx.distributed:
        del kl, vl
        edist.release_peer_buffers()
    torch.cuda.empty_cache()
    return row




def sweep_block(args, ctx, elsa, hl, spec_peak):
    """N = 1 kernel-only sweep: CUDA-graph replays, L2 flushed between them."""
    torch, dev, stream = ctx.torch, ctx.dev, ctx.stream
    q, k, v = hl["q"], hl["k"], hl["v"]
    B, H, n = q.shape[0], q.shape[1], q.shape[2]
    fl = hl["fl"]
    sweep = []
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
    gen = torch.Generator(device=dev)
    gen.manual_seed(16)
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
    del flush
    return sweep


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    ctx = Ctx(args)
    torch = ctx.torch
    import paper_2604_23798_b200 as elsa
    from paper_2604_23798_b200 import dist as edist

    world, rank = ctx.world, ctx.rank
    peaks = measured_peaks()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    spec_peak = SMS * FFMA_LANES * 2 * fmax * 1e6 / 1e12

    hl = headline(args, ctx, elsa, edist)
    strong = None
    if ctx.distributed and args.shard == "q" and world > 1:
        strong = strong_c3(args, ctx, elsa, edist, hl)
    e2e = None if args.no_e2e else e2e_block(args, ctx, elsa, hl)

    # ---- roofline: FFMA peak (spec clock) and the K4 microbenchmark ----
    k4 = None
    try:
        k4 = elsa.ffma_peak_tflops(ctx.dev)
    except Exception:  # noqa: BLE001
        k4 = None
    per_gpu = hl["value"] / world
    traffic, traffic_workload = ncu_traffic()
    B1 = args.batch
    roofline = {
        "bound": "ffma", "achieved": per_gpu, "peak": spec_peak, "unit": "TFLOP/s",
        "frac": per_gpu / spec_peak,
        "peak_source": f"148 SM x 128 FP32 lanes x 2 x {fmax:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
        "k4_ffma_measured": k4, "frac_of_k4": (per_gpu / k4) if k4 else None,
        "traffic": traffic, "traffic_workload": traffic_workload,
        # the K/V (and Q, Y) streams: DRAM bytes of the ncu capture over this
        # run's kernel time (the north star's HBM GB/s evidence; far below the
        # HBM roofline: the kernel is FFMA-bound at n/4 flop per byte)
        "hbm_gbs": (traffic / (hl["ms"] * 1e-3) / 1e9) if traffic else None,
        "hbm_peak_gbs": float(peaks.get("hbm_gbs") or 6650.0),
        "hbm_peak_source": "MEASURED_PEAKS hbm_gbs" if peaks.get("hbm_gbs") else
                           "fallback 6.65 TB/s (B200_PROFILING.md)",
        "algorithmic_flops_per_launch": flops(B1, args.heads, args.n, args.n),
        "algorithmic_bytes_per_launch": 4 * B1 * args.heads * (args.n * 64 * 3 + args.n * 64),
        "kernel": "elsa::fwd_f32_kernel (" + hl["plan"] + ")",
        "measurement": "CUDA events on the launching stream around the K timed steps (max over "
                       "ranks); one kernel launch per GPU per step at this shape",
    }

    sweep = []
    if not args.no_sweep and not ctx.distributed:
        sweep = sweep_block(args, ctx, elsa, hl, spec_peak)

    # free the headline tensors before the long-context problems (C5: 8 GiB)
    q_shape = tuple(hl["q"].shape)
    for key in ("q", "k", "v"):
        hl.pop(key)
    hl["state"].clear()
    torch.cuda.empty_cache()
    longc = long_context(args, ctx, elsa, edist, spec_peak)

    # ---- CPU baseline: the reference's algorithm on the host cores (rank 0, N=1) ----
    cpu = None
    if rank == 0 and not ctx.distributed and not args.no_cpu_baseline:
        n, H, B = args.n, args.heads, args.batch
        workers = _cpu_workers(args, _lane_gb(n))
        tiles = args.cpu_sample_tiles or workers
        val, secs, desc = cpu_baseline_sample(n, H, B, tiles, workers)
        full_workers = _cpu_workers(args, _lane_gb(2048))
        cpu = {"value": val, "unit": "TFLOP/s", "cores": workers, "kind": "port",
               "sample": desc, "seconds": secs, **host_info(),
               "full_small_configs": cpu_full_configs(full_workers)}

    Bg = hl["Bg"]
    if rank == 0:
        if ctx.distributed and args.shard == "q":
            workload = (f"C3 FP32 attention B{Bg} H{args.heads} n{args.n} d64 dv64: one "
                        f"B{args.batch} H{args.heads} n{args.n} problem per GPU, (b, h, q) row "
                        f"slices, no exchange")
            par = f"batch x heads row slices over {world} GPUs (query-sharded)"
        elif ctx.distributed:
            workload = (f"C3 FP32 attention B{Bg} H{args.heads} n{args.n} d64 dv64, KV-sharded "
                        f"over {world} GPUs ({hl['chunks']} chunks)")
            par = f"kv-shard{world}"
        else:
            workload = f"C3 FP32 attention B{Bg} H{args.heads} n{args.n} d64 dv64"
            par = "single GPU"
        line = {
            "metric": METRIC, "value": hl["value"], "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": hl["warmup"], "ms_per_step": hl["ms"],
            "higher_is_better": True,
            "scaling": "weak" if (ctx.distributed and args.shard == "q") or world == 1
                       else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic N(0,1) Q/K/V (torch.randn), resident in HBM",
            "config": {"workload": workload, "B": Bg, "H": args.heads, "n": args.n, "d": 64,
                       "dv": 64, "shape": list(q_shape),
                       "l2": "inputs 3x%.0f MB per GPU > 126 MB L2 (no L2 reuse across steps); "
                             "the sweep flushes L2 (256 MB write) between timed iterations"
                             % (args.batch * args.heads * args.n * 64 * 4 / 1e6),
                       "parallelism": par},
            "parity": hl["parity"],
            "e2e": e2e, "gpu_launches": hl["launches"], "clocks": hl["clocks"],
            "roofline": roofline, "strong": strong, "long_context": longc, "comm": ctx.comm,
            "cpu_baseline": cpu, "sweep": sweep,
        }
        print(json.dumps(line), flush=True)
    if ctx.distributed:
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
