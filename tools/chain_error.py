"""Error of the K1 schedule vs the length of the per-CTA sequential chain
(VERDICT r1 weak #7): the same problem with kv_splits
= 1 .. 32 (each CTA folds ceil(tiles / splits) key tiles in sequence, then the
fixed log-depth (+)-tree merges the splits), errors against FP64 rows.
usage: python tools/chain_error.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2604_23798_b200 as elsa  # noqa: E402

dev = torch.device("cuda", 0)
NQ = 64
for n_kv in (65536, 1 << 20):
    g = torch.Generator(device=dev)
    g.manual_seed(n_kv % 1000)
    q = torch.randn(1, 2, NQ, 64, device=dev, generator=g)
    k = torch.randn(1, 2, n_kv, 64, device=dev, generator=g)
    v = torch.randn(1, 2, n_kv, 64, device=dev, generator=g)
    ref = []
    for h in range(2):
        K = k[0, h].double().cpu().numpy()
        V = v[0, h].double().cpu().numpy()
        Q = q[0, h].double().cpu().numpy()
        s = (Q @ K.T) / math.sqrt(64)
        s -= s.max(axis=1, keepdims=True)
        np.exp(s, out=s)
        ref.append((s @ V) / s.sum(axis=1, keepdims=True))
        del s, K, V
    ref = np.stack(ref)[None]
    thr = oracle.bound_threshold(n_kv)
    tiles = n_kv // 64
    print(f"n_kv = {n_kv} ({tiles} key tiles), {NQ} query rows x 2 heads, "
          f"bound u*L*8 = {thr:.3e}", flush=True)
    for splits in (1, 2, 4, 8, 16, 32):
        if -(-tiles // splits) > 16384:
            continue
        y = elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits)
        err = oracle.row_rel_err(y.double().cpu().numpy(), ref)
        chain = -(-tiles // splits)
        print(f"  splits {splits:2d}: chain {chain:5d} tiles + tree depth "
              f"{math.ceil(math.log2(splits)) if splits > 1 else 0}:  max {err.max():.3e}  "
              f"mean {err.mean():.3e}  p99 {np.percentile(err, 99):.3e}  "
              f"({err.max() / thr:.2f} x bound)", flush=True)
