"""The host-buffer entry point (elsa_fwd_f32_host / attention_from_host):
the reference's scan_forward takes and returns host arrays
(engine.py:385-427); this path copies them in and out with the copies
pipelined under the kernels. Its Y must be bitwise identical to the device
entry point's with the same plan, and within the FP64 bound."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_23798_b200 as elsa  # noqa: E402

DEV = torch.device("cuda", 0)


def _inputs(B, H, n_q, n_kv, d=64, dv=64, seed=0, pin=True):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(B, H, n_q, d, generator=g)
    k = torch.randn(B, H, n_kv, d, generator=g)
    v = torch.randn(B, H, n_kv, dv, generator=g)
    if pin:
        q, k, v = q.pin_memory(), k.pin_memory(), v.pin_memory()
    return q, k, v


@pytest.mark.parametrize("B,H,n_q,n_kv,splits", [
    (1, 16, 1024, 1024, 0),   # 16 groups of one head
    (3, 7, 300, 517, 0),      # 21 heads -> 11 groups of 2 (ragged last group), ragged n
    (1, 2, 2048, 2048, 0),    # auto splits > 1: per-stream split workspace
    (2, 5, 256, 640, 3),      # explicit splits
    (1, 1, 1, 1, 0),          # single token
])
def test_host_matches_device_bitwise(B, H, n_q, n_kv, splits):
    q, k, v = _inputs(B, H, n_q, n_kv)
    y_host = elsa.attention_from_host(q, k, v, kv_splits=splits, check_numerics=True)
    assert y_host.device.type == "cpu"
    y_dev = elsa.scaled_dot_product_attention(q.to(DEV), k.to(DEV), v.to(DEV), kv_splits=splits,
                                              check_numerics=True).cpu()
    assert torch.equal(y_host, y_dev)


def test_host_pageable_numpy_and_out_within_bound():
    Q, K, V = oracle.generate(11, "regular", b=2, h=3, n=384, d=64, d_v=64, dtype=np.float32)
    y = elsa.attention_from_host(Q, K, V)  # pageable numpy inputs
    ref = oracle.naive_attention(Q, K, V)
    err = oracle.row_rel_err(y.numpy(), ref)
    assert err.max() <= oracle.bound_threshold(384)
    out = torch.empty(2, 3, 384, 64).pin_memory()
    y2 = elsa.attention_from_host(torch.from_numpy(Q).pin_memory(), torch.from_numpy(K),
                                  torch.from_numpy(V), out=out)
    assert y2 is out and torch.equal(out, y)


def test_host_head_dims_and_scale():
    q, k, v = _inputs(1, 3, 200, 333, d=24, dv=40, seed=3)
    y = elsa.attention_from_host(q, k, v, scale=-0.3)
    ref = oracle.naive_attention(q.numpy(), k.numpy(), v.numpy(), scale=-0.3)
    assert oracle.row_rel_err(y.numpy(), ref).max() <= oracle.bound_threshold(333)


def test_host_back_to_back_calls_reuse_workspace():
    # async calls on one stream: the second call's copies must not overwrite
    # device inputs the first call's kernels still read
    a = _inputs(1, 8, 2048, 2048, seed=5)
    b = _inputs(1, 8, 2048, 2048, seed=6)
    ya = torch.empty(1, 8, 2048, 64).pin_memory()
    yb = torch.empty(1, 8, 2048, 64).pin_memory()
    elsa.attention_from_host(*a, out=ya, sync=False)
    elsa.attention_from_host(*b, out=yb, sync=False)
    torch.cuda.synchronize()
    for (q, k, v), y in ((a, ya), (b, yb)):
        ref = elsa.scaled_dot_product_attention(q.to(DEV), k.to(DEV), v.to(DEV)).cpu()
        assert torch.equal(y, ref)


def test_host_numerical_error_and_rejections():
    q, k, v = _inputs(1, 1, 64, 64, pin=False)
    k[0, 0, 3, 0] = float("inf")
    with pytest.raises(elsa.NumericalError):
        elsa.attention_from_host(q, k, v, check_numerics=True)
    with pytest.raises(elsa.ShapeError):
        elsa.attention_from_host(q.double(), k, v)
    with pytest.raises(elsa.ShapeError):
        elsa.attention_from_host(q.to(DEV), k, v)
