"""Kernel time of small shapes (C1, 1K, BERT, 2K) per kv split request (0 = planner), CUDA-graph replays, L2 flushed."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_23798_b200 as elsa
dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
def time_fn(fn, iters=50):
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
    ts.sort(); return ts[len(ts)//2]
for (B,H,n) in ((1,1,1024),(1,16,1024),(8,12,512),(1,16,2048)):
    q,k,v=(torch.randn(B,H,n,64,device=dev) for _ in range(3))
    fl=4.0*B*H*n*n*64
    row=[]
    for sp in (0,1,2,3,4,6,8,12,16):
        ms=time_fn(lambda: elsa.scaled_dot_product_attention(q,k,v,kv_splits=sp))
        row.append(f"s{sp}:{ms*1e3:.1f}us")
    print(f"B{B} H{H} n{n}: "+" ".join(row), flush=True)
