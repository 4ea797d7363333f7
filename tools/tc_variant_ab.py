"""A/B of K5 (tcgen05 FP16/BF16) compile variants on one box: for every
build/var_<name>.so given, time BF16/FP16 at n = 4K/16K (CUDA-graph replays, L2
flushed) and the max per-row error vs FP64 at n = 2K next to PyTorch's own
16-bit SDPA error. Each variant runs in its own process (ELSA_LIB_PATH).

usage: python tools/tc_variant_ab.py build/var_a.so build/var_b.so ..."""
import os
import subprocess
import sys

CHILD = r'''
import os, sys, math, torch
sys.path.insert(0, os.getcwd())
import paper_2604_23798_b200 as elsa
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def time_fn(fn, iters=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s): fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); g.replay(); b.record(s); b.synchronize()
            ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]
out = []
for dt in (torch.bfloat16, torch.float16):
    for n in (4096, 16384):
        q, k, v = (torch.randn(1, 16, n, 64, device=dev, dtype=dt) for _ in range(3))
        ms = time_fn(lambda: elsa.scaled_dot_product_attention(q, k, v))
        out.append(f"{str(dt)[6:]} n{n} {4.0*16*n*n*64/ms/1e9:6.1f}")
    torch.manual_seed(1)
    q, k, v = (torch.randn(1, 4, 2048, 64, device=dev) for _ in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(q.double(), k.double(), v.double())
    def err(y):
        y = y.double()
        return ((y - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
    e_ours = err(elsa.scaled_dot_product_attention(q.to(dt), k.to(dt), v.to(dt)))
    e_t = err(torch.nn.functional.scaled_dot_product_attention(q.to(dt), k.to(dt), v.to(dt)))
    out.append(f"{str(dt)[6:]} err {e_ours:.2e} (torch {e_t:.2e})")
print(" | ".join(out), flush=True)
'''

for so in sys.argv[1:]:
    env = dict(os.environ, ELSA_LIB_PATH=os.path.abspath(so))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                       timeout=600)
    name = os.path.basename(so)
    print(f"{name:24s} {r.stdout.strip() or r.stderr.strip().splitlines()[-1]}", flush=True)
