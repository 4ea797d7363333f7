"""Time the §8f row-3 path on the GPU: per-key-block states for every query
(elsa_blockwise_f32) and the reference-shaped two-pass block combine with
prefixes (elsa_block_scan_f32), CUDA-graph replays, L2 flushed between."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t_graph(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            ts.append((a, b))
        torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) for x, y in ts)
    return v[len(v) // 2]


for (B, H, n, blk) in [(1, 16, 4096, 128), (1, 16, 16384, 1024), (8, 12, 512, 128)]:
    q, k, v = (torch.randn(B, H, n, 64, device=dev) for _ in range(3))
    states = elsa.blockwise_states(q, k, v, block_size=blk)
    ms_b = t_graph(lambda: elsa.blockwise_states(q, k, v, block_size=blk))
    ms_s = t_graph(lambda: elsa.inter_block_combine(*states, return_prefixes=True))
    fl = 2.0 * B * H * n * n * 128
    nb = -(-n // blk)
    state_bytes = B * H * n * nb * 66 * 4
    print(f"B{B} H{H} n{n} block {blk}: blockwise_states {ms_b:.3f} ms ({fl / ms_b / 1e9:.1f} TFLOP/s, "
          f"{state_bytes / 1e9:.2f} GB of states); block combine+prefixes {ms_s:.3f} ms "
          f"({3 * state_bytes / ms_s / 1e6:.0f} GB/s of state traffic)", flush=True)
