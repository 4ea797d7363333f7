"""Time K5 (tcgen05 FP16/BF16) against torch SDPA (flash backend) on the same
inputs; CUDA-graph replays, L2 flushed between, events on the capture stream."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2604_23798_b200 as elsa

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def time_fn(fn, iters=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(iters):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            b.synchronize()
            tot += a.elapsed_time(b)
    return tot / iters


D = int(os.environ.get("D", "64"))  # head width (64, or up to 128: the D = 128 kernel)
for dt in (torch.bfloat16, torch.float16):
    for (B, H, n) in [(1, 16, 1024), (1, 16, 4096), (1, 16, 16384), (8, 12, 512), (1, 16, 65536)]:
        q, k, v = (torch.randn(B, H, n, D, device=dev, dtype=dt) for _ in range(3))
        flops = 4.0 * B * H * n * n * D
        ms = time_fn(lambda: elsa.scaled_dot_product_attention(q, k, v))
        mt = time_fn(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
        print(f"{str(dt):15s} d{D} B{B} H{H} n{n:6d}: elsa {ms:8.3f} ms {flops/ms/1e9:7.1f} TF/s | "
              f"torch {mt:8.3f} ms {flops/mt/1e9:7.1f} TF/s", flush=True)
