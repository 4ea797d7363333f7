"""K1 with the thread-block-cluster split merge (fwd_f32_kernel<..., CL>):
the kv splits of one query tile merge over distributed shared memory inside
the launch. Same partial states, same fixed tree (monoid.py:234-265), same
arithmetic as the two-launch path (K1 partial states -> K2), so the result
must be BITWISE equal to it for every split count, and within the FP64 bound."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_23798_b200 as elsa  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture
def cluster_mode():
    yield elsa.attention.set_cluster_mode
    elsa.attention.set_cluster_mode(1)


@pytest.mark.parametrize("B,H,n_q,n_kv", [(1, 1, 1024, 1024), (8, 12, 512, 512), (1, 3, 333, 1000),
                                          (2, 2, 64, 4096), (1, 1, 1, 700), (1, 2, 200, 65)])
@pytest.mark.parametrize("splits", [2, 3, 4, 8, 11, 16])
def test_cluster_merge_bitwise_equals_two_launch_path(cluster_mode, B, H, n_q, n_kv, splits):
    rng = np.random.default_rng(B * 100 + n_q + splits)
    Q = rng.standard_normal((B, H, n_q, 64)).astype(np.float32)
    K = rng.standard_normal((B, H, n_kv, 64)).astype(np.float32)
    V = rng.standard_normal((B, H, n_kv, 64)).astype(np.float32)
    q, k, v = (torch.from_numpy(x).to(DEV) for x in (Q, K, V))
    cluster_mode(2)
    plan = elsa.describe_plan(q, k, v, splits)
    ws = elsa.attention.workspace_bytes(q, k, v, splits)
    y_clu = elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits, check_numerics=True)
    cluster_mode(0)
    plan0 = elsa.describe_plan(q, k, v, splits)
    y_k2 = elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits, check_numerics=True)
    assert "cluster_merge" not in plan0
    n_split = int(plan.split("kv_splits=")[1].split()[0])
    if n_split > 1:
        assert "cluster_merge=dsmem" in plan, plan
        assert ws == 0
    assert torch.equal(y_clu, y_k2), (plan, (y_clu - y_k2).abs().max().item())
    ref = oracle.naive_attention_rows_fp64(Q, K, V)
    err = oracle.row_rel_err(y_clu.cpu().numpy(), ref)
    assert err.max() <= oracle.bound_threshold(n_kv)


def test_cluster_plan_single_launch_no_workspace(cluster_mode):
    """C1 (B1 H1 n1024): the auto plan merges its splits inside one launch
    and needs no split workspace."""
    q = torch.randn(1, 1, 1024, 64, device=DEV)
    cluster_mode(1)
    plan = elsa.describe_plan(q, q, q)
    if "cluster_merge" in plan:
        assert elsa.attention.workspace_bytes(q, q, q) == 0
        elsa.scaled_dot_product_attention(q, q, q)
        assert elsa.last_launch_count() == 1
    cluster_mode(2)
    y = elsa.scaled_dot_product_attention(q, q, q, kv_splits=8)
    assert elsa.last_launch_count() == 1
    cluster_mode(0)
    y0 = elsa.scaled_dot_product_attention(q, q, q, kv_splits=8)
    assert elsa.last_launch_count() == 2
    assert torch.equal(y, y0)


def test_cluster_strided_output_and_negative_scale(cluster_mode):
    g = torch.Generator(device=DEV)
    g.manual_seed(9)
    q = torch.randn(1, 2, 300, 64, device=DEV, generator=g)
    k = torch.randn(1, 2, 900, 64, device=DEV, generator=g)
    v = torch.randn(1, 2, 900, 64, device=DEV, generator=g)
    out = torch.empty(1, 300, 2, 64, device=DEV).transpose(1, 2)   # head-strided Y
    cluster_mode(2)
    elsa.scaled_dot_product_attention(q, k, v, kv_splits=4, out=out, scale=-0.3)
    cluster_mode(0)
    ref = elsa.scaled_dot_product_attention(q, k, v, kv_splits=4, scale=-0.3)
    assert torch.equal(out, ref)


# ---- tail split (last wave's units as key pieces + K2 over their rows) ----

@pytest.mark.parametrize("shape,mode", [((8, 12, 512), 1), ((8, 12, 512), 3), ((8, 16, 512), 2),
                                        ((16, 12, 500), 5)])
def test_tail_split_parity_and_full_units_bitwise(shape, mode):
    """Tail-split plans (ELSA_TAIL / set_tail_mode): every row within the
    reference bound vs FP64, and the rows of the whole units (before the
    tail) bitwise equal to the plan without the tail split (same kernel code
    for them)."""
    b, h, n = shape
    rng = np.random.default_rng(b * 1000 + n)
    Q, K, V = (rng.standard_normal((b, h, n, 64)).astype(np.float32) for _ in range(3))
    q, k, v = (torch.from_numpy(x).to(DEV) for x in (Q, K, V))
    try:
        elsa.attention.set_tail_mode(0)
        y0 = elsa.scaled_dot_product_attention(q, k, v)
        elsa.attention.set_tail_mode(mode)
        plan = elsa.describe_plan(q, k, v)
        y1 = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
    finally:
        elsa.attention.set_tail_mode(1)
    assert "tail_split=" in plan, plan
    first = int(plan.split("units>=")[1].rstrip(")"))
    tq = int(plan.split("tq=")[1].split()[0])
    qt = -(-n // tq)
    row0 = (first // qt) * n + (first % qt) * tq
    f0, f1 = y0.reshape(-1, 64), y1.reshape(-1, 64)
    assert torch.equal(f0[:row0], f1[:row0])
    ref = oracle.naive_attention(Q.astype(np.float64), K.astype(np.float64), V.astype(np.float64))
    err = oracle.row_rel_err(y1.cpu().numpy(), ref)
    assert err.max() <= oracle.bound_threshold(n), err.max()
