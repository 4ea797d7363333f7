import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2604_23798_b200 as elsa, oracle
for (b, h, n) in [(8, 12, 512), (1, 16, 4096), (4, 12, 512)]:
    g = torch.Generator(device='cuda'); g.manual_seed(n + b)
    q, k, v = (torch.randn(b, h, n, 64, device='cuda', generator=g) for _ in range(3))
    y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
    Q, K, V = (t.double().cpu().numpy() for t in (q, k, v))
    ref = oracle.naive_attention(Q, K, V)
    err = oracle.row_rel_err(y.double().cpu().numpy(), ref)
    print(b, h, n, elsa.describe_plan(q, k, v), 'max err', err.max(), 'bound', oracle.bound_threshold(n))
