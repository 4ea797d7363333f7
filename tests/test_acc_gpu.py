"""The long-chain K1 kernel (`w8r8acc`, fwd_f32_kernel<..., ACC = true>):
two-level W accumulation (each key tile's P V in a fresh accumulator, folded
into the running W once per tile).

Gate: the reference's per-row bound u * L(n, 128) * 8 (verify.py:339-343)
against the FP64 oracle (oracles.py:74-104 restated in ``oracle``), on
ragged shapes, kv splits, partial states and strided inputs; and the point of
the kernel: over a long sequential chain its error is well below the
one-level kernel's.
"""

import math

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_23798_b200 as elsa  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture
def acc():
    elsa.attention.force_config("w8r8acc")
    yield
    elsa.attention.force_config(None)


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


@pytest.mark.parametrize("n_q,n_kv,splits", [(1, 1, 0), (77, 300, 0), (128, 1000, 0),
                                             (300, 4097, 3), (513, 2048, 0), (64, 8192, 7)])
def test_acc_parity_vs_fp64(acc, n_q, n_kv, splits):
    rng = np.random.default_rng(n_q * 7 + n_kv)
    Q = rng.standard_normal((2, 3, n_q, 64)).astype(np.float32)
    K = rng.standard_normal((2, 3, n_kv, 64)).astype(np.float32)
    V = rng.standard_normal((2, 3, n_kv, 64)).astype(np.float32)
    assert elsa.describe_plan(gpu(Q), gpu(K), gpu(V), splits).startswith("w8r8acc")
    y = elsa.scaled_dot_product_attention(gpu(Q), gpu(K), gpu(V), kv_splits=splits,
                                          check_numerics=True).cpu().numpy()
    ref = oracle.naive_attention(Q.astype(np.float64), K.astype(np.float64),
                                 V.astype(np.float64))
    err = oracle.row_rel_err(y, ref)
    assert err.max() <= oracle.bound_threshold(n_kv), err.max()
    if n_kv == 1:
        assert np.array_equal(y, np.broadcast_to(V, y.shape))  # n = 1 returns v exactly


def test_acc_partial_states_and_strided(acc):
    rng = np.random.default_rng(3)
    base = gpu(rng.standard_normal((1, 2, 700, 80)).astype(np.float32))
    q = base[..., 3:67]          # 4-byte-aligned, row-strided: the copy engine
    k = gpu(rng.standard_normal((1, 2, 900, 64)).astype(np.float32))
    v = gpu(rng.standard_normal((1, 2, 900, 64)).astype(np.float32))
    y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
    Q64, K64, V64 = (t.double().cpu().numpy() for t in (q, k, v))
    ref = oracle.naive_attention(Q64, K64, V64)
    assert oracle.row_rel_err(y.cpu().numpy(), ref).max() <= oracle.bound_threshold(900)
    m0, S0, W0 = elsa.partial_states(q, k, v, 0, 450)
    m1, S1, W1 = elsa.partial_states(q, k, v, 450, 900)
    y2 = elsa.merge_states(torch.stack([m0, m1]), torch.stack([S0, S1]), torch.stack([W0, W1]))
    assert oracle.row_rel_err(y2.cpu().numpy(), ref).max() <= oracle.bound_threshold(900)


def test_acc_long_chain_error_below_one_level_kernel():
    """64 query rows x 2 heads against 2^18 keys in ONE split (a 4096-tile
    sequential chain per CTA): the two-level kernel's max row error must be
    at most half the one-level kernel's (measured ~7x lower at 1024-16384
    tiles, profiles/round2_chain_error_acc.txt), and within the bound."""
    n_kv = 1 << 18
    g = torch.Generator(device=DEV)
    g.manual_seed(18)
    q = torch.randn(1, 2, 64, 64, device=DEV, generator=g)
    k = torch.randn(1, 2, n_kv, 64, device=DEV, generator=g)
    v = torch.randn(1, 2, n_kv, 64, device=DEV, generator=g)
    ref = []
    for h in range(2):
        K = k[0, h].double().cpu().numpy()
        s = (q[0, h].double().cpu().numpy() @ K.T) / math.sqrt(64)
        s -= s.max(axis=1, keepdims=True)
        np.exp(s, out=s)
        ref.append((s @ v[0, h].double().cpu().numpy()) / s.sum(axis=1, keepdims=True))
    ref = np.stack(ref)[None]
    errs = {}
    try:
        for cfg in ("w8r8", "w8r8acc"):
            elsa.attention.force_config(cfg)
            y = elsa.scaled_dot_product_attention(q, k, v, kv_splits=1)
            errs[cfg] = oracle.row_rel_err(y.double().cpu().numpy(), ref).max()
    finally:
        elsa.attention.force_config(None)
    assert errs["w8r8acc"] <= oracle.bound_threshold(n_kv)
    assert errs["w8r8acc"] <= 0.5 * errs["w8r8"], errs


def test_planner_uses_acc_kernel_past_the_one_level_cap():
    """Past kMaxSplits x 1024 tiles the one-level kernel would exceed its
    chain cap; the planner picks the two-level kernel (cap 16384 tiles)."""
    q = torch.empty(1, 1, 1024, 64, device=DEV)
    kk = torch.empty(1, 1, 1, 64, device=DEV).expand(1, 1, 1 << 22, 64)
    plan = elsa.describe_plan(q, kk, kk)
    assert plan.startswith("w8r8acc") and "chain_tiles" not in plan, plan
