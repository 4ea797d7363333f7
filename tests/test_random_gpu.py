"""Randomised shapes through every K1 plan family (GPU): the planner's choice,
forced tail splits, the two-level-accumulator kernel, cluster merges and
explicit kv splits, each checked row by row against the FP64 oracle
(oracles.py:74-104) within the reference bound u * L(n_kv, 128) * 8
(verify.py:339-343). Shapes are ragged (n_q != n_kv, tails of every size,
d and dv below 64) and the inputs strided where drawn so."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_23798_b200 as elsa  # noqa: E402

DEV = torch.device("cuda", 0)
MODES = ["auto", "tail3", "acc", "cluster", "splits5"]


def _draw(seed):
    rng = np.random.default_rng(seed)
    B = int(rng.integers(1, 4))
    H = int(rng.integers(1, 7))
    n_q = int(rng.integers(1, 700))
    n_kv = int(rng.integers(1, 900))
    d = int(rng.choice([8, 16, 32, 48, 64]))
    dv = int(rng.choice([4, 16, 33, 64]))
    strided = bool(rng.integers(0, 2))
    return rng, B, H, n_q, n_kv, d, dv, strided


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("mode", MODES)
def test_random_shapes_all_plan_families(seed, mode):
    rng, B, H, n_q, n_kv, d, dv, strided = _draw(1000 + seed)
    Q = rng.standard_normal((B, H, n_q, d)).astype(np.float32)
    K = rng.standard_normal((B, H, n_kv, d)).astype(np.float32)
    V = rng.standard_normal((B, H, n_kv, dv)).astype(np.float32)
    if strided:  # row-strided views of wider buffers
        qb = torch.zeros(B, H, n_q, d + 8, device=DEV)
        qb[..., :d] = torch.from_numpy(Q).to(DEV)
        q = qb[..., :d]
    else:
        q = torch.from_numpy(Q).to(DEV)
    k, v = torch.from_numpy(K).to(DEV), torch.from_numpy(V).to(DEV)
    splits = 0
    try:
        if mode == "tail3":
            elsa.attention.set_tail_mode(3)
        elif mode == "acc":
            elsa.attention.force_config("w8r8acc")
        elif mode == "cluster":
            elsa.attention.set_cluster_mode(2)
            splits = 3
        elif mode == "splits5":
            splits = 5
        y = elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits, check_numerics=True)
        plan = elsa.describe_plan(q, k, v, splits)
    finally:
        elsa.attention.set_tail_mode(1)
        elsa.attention.force_config(None)
        elsa.attention.set_cluster_mode(1)
    ref = oracle.naive_attention(Q.astype(np.float64), K.astype(np.float64),
                                 V.astype(np.float64))
    # very narrow V rows can nearly cancel: error relative to the magnitudes mixed
    err = oracle.row_err_conditioned(y.cpu().numpy(), Q, K, V, ref=ref) \
        if dv <= 4 else oracle.row_rel_err(y.cpu().numpy(), ref)
    assert err.max() <= oracle.bound_threshold(n_kv), (plan, err.max())
