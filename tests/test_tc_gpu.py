"""K5: the FP16 / BF16 variant on the tcgen05 tensor cores,
checked against the FP64 oracle on the same (16-bit-rounded) inputs. The
16-bit P operand and 16-bit output bound the accuracy; the gate is 2x the
error of PyTorch's own 16-bit SDPA on the same inputs (plus an absolute floor
at the output format's unit roundoff)."""

import math

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2604_23798_b200 as elsa  # noqa: E402

DEV = torch.device("cuda", 0)


def _check(dtype, B, H, n_q, n_kv, seed, scale=None, d=64, dv=64):
    g = torch.Generator(device=DEV)
    g.manual_seed(seed)
    q = torch.randn(B, H, n_q, d, device=DEV, generator=g).to(dtype)
    k = torch.randn(B, H, n_kv, d, device=DEV, generator=g).to(dtype)
    v = torch.randn(B, H, n_kv, dv, device=DEV, generator=g).to(dtype)
    y = elsa.scaled_dot_product_attention(q, k, v, scale=scale, check_numerics=True)
    assert y.dtype == dtype and y.shape == (B, H, n_q, dv)
    ref = oracle.naive_attention(*(t.double().cpu().numpy() for t in (q, k, v)), scale=scale)
    ours = oracle.row_rel_err(y.double().cpu().numpy(), ref)
    # PyTorch's 16-bit SDPA returns NaN for a negative scale: give it the
    # sign on Q instead (the same product)
    qs, sc = (-q, -scale) if scale is not None and scale < 0 else (q, scale)
    theirs = oracle.row_rel_err(torch.nn.functional.scaled_dot_product_attention(
        qs, k, v, scale=sc).double().cpu().numpy(), ref)
    u = 2.0 ** -8 if dtype == torch.bfloat16 else 2.0 ** -11
    assert np.percentile(ours, 99) <= max(2 * np.percentile(theirs, 99), u), (
        np.percentile(ours, 99), np.percentile(theirs, 99))
    assert ours.max() <= max(2 * theirs.max(), 2 * u)
    return ours.max()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("B,H,n_q,n_kv", [(1, 2, 128, 128), (1, 4, 1024, 1024), (2, 3, 200, 333),
                                          (1, 1, 1, 1), (1, 2, 129, 4096)])
def test_tc_matches_fp64(dtype, B, H, n_q, n_kv):
    _check(dtype, B, H, n_q, n_kv, seed=n_q * 31 + n_kv)


def test_tc_negative_scale_and_determinism():
    _check(torch.bfloat16, 1, 2, 256, 256, seed=3, scale=-0.2)
    q = torch.randn(1, 2, 300, 64, device=DEV, dtype=torch.bfloat16)
    a = elsa.scaled_dot_product_attention(q, q, q)
    b = elsa.scaled_dot_product_attention(q, q, q)
    assert torch.equal(a, b)


def test_tc_rejects_other_head_dims():
    q = torch.randn(1, 1, 16, 136, device=DEV, dtype=torch.bfloat16)
    with pytest.raises(elsa.ShapeError):
        elsa.scaled_dot_product_attention(q, q, q)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("d,dv", [(32, 32), (16, 64), (64, 16), (40, 24), (8, 8), (60, 36),
                                  (3, 5), (64, 1), (128, 128), (96, 80), (128, 64), (64, 128),
                                  (100, 128), (72, 8)])
def test_tc_narrow_heads(dtype, d, dv):
    # d, dv < 64: the 64-wide TMA boxes zero-fill past the row (rows not a
    # multiple of 8 elements are first copied into padded rows); Y rows narrower
    # than 64 are stored element-wise
    if dv <= 8:  # narrow rows can cancel to ~0: absolute tolerance against FP32
        g = torch.Generator(device=DEV)
        g.manual_seed(d)
        q, k = (torch.randn(1, 2, 300, d, device=DEV, generator=g).to(dtype) for _ in range(2))
        v = torch.randn(1, 2, 300, dv, device=DEV, generator=g).to(dtype)
        y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
        ref = elsa.scaled_dot_product_attention(q.float(), k.float(), v.float())
        assert y.shape == (1, 2, 300, dv)
        assert torch.allclose(y.float(), ref, atol=2e-2, rtol=2e-2)
        return
    _check(dtype, 1, 3, 300, 333, seed=d * 100 + dv, d=d, dv=dv)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_tc_two_tile_ctas_ragged(dtype):
    # >= one wave of two-query-tile CTAs: the ping-pong (two softmax warpgroups)
    # kernel, with ragged n_q (partial second tile) and a ragged key tail
    _check(dtype, 2, 8, 4096 + 77, 1000, seed=41)


def test_tc_deferred_anchor_moves():
    # logits that grow along the key axis: every tile raises the row maximum
    # by more than the 2^8 hysteresis, so the W rows in TMEM are rescaled
    # (the rare path of the deferred anchor) tile after tile
    g = torch.Generator(device=DEV)
    g.manual_seed(7)
    B, H, n = 2, 8, 4096
    q = torch.randn(B, H, n, 64, device=DEV, generator=g)
    k = torch.randn(B, H, n, 64, device=DEV, generator=g)
    ramp = torch.linspace(0.2, 3.0, n, device=DEV).view(1, 1, n, 1)
    k = (k * ramp + ramp * 2.0).to(torch.bfloat16)
    q = (q.abs() + 0.5).to(torch.bfloat16)
    v = torch.randn(B, H, n, 64, device=DEV, generator=g).to(torch.bfloat16)
    y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
    ref = oracle.naive_attention(*(t.double().cpu().numpy() for t in (q, k, v)))
    ours = oracle.row_rel_err(y.double().cpu().numpy(), ref)
    theirs = oracle.row_rel_err(torch.nn.functional.scaled_dot_product_attention(
        q, k, v).double().cpu().numpy(), ref)
    assert np.percentile(ours, 99) <= max(2 * np.percentile(theirs, 99), 2.0 ** -8)
    assert ours.max() <= max(2 * theirs.max(), 2.0 ** -7)


@pytest.mark.parametrize("seed", range(10))
def test_tc_random_geometry_fuzz(seed):
    # seeded random batch / heads / ragged lengths / scale sign for the 16-bit
    # path (one- and two-tile CTAs, tail tiles) against FP64
    rng = np.random.default_rng(7000 + seed)
    dtype = torch.bfloat16 if seed % 2 else torch.float16
    B, H = int(rng.integers(1, 4)), int(rng.integers(1, 6))
    n_q, n_kv = int(rng.integers(1, 900)), int(rng.integers(1, 900))
    scale = None if seed % 3 else float(rng.choice([-1, 1]) * rng.uniform(0.05, 0.2))
    _check(dtype, B, H, n_q, n_kv, seed, scale=scale)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_tc_d128_long_and_ragged(dtype):
    # the D = 128 kernel (two 64-element column blocks per row, W 128 columns
    # in TMEM, 2-stage ring) over many key tiles with ragged tails
    _check(dtype, 2, 3, 1000 + 37, 2048 + 77, seed=5, d=128, dv=128)
    _check(dtype, 1, 2, 300, 700, seed=6, scale=-0.09, d=128, dv=128)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_tc_d128_two_tile_ctas_aliased_p(dtype):
    # >= one wave of two-query-tile CTAs at d = 128: P written over S in TMEM
    # and S_g(t+1) issued only after P_g(t) V (ragged rows and key tail)
    _check(dtype, 1, 16, 2560 + 33, 300 + 5, seed=17, d=128, dv=128)
    _check(dtype, 2, 8, 2560, 1000, seed=18, scale=-0.1, d=112, dv=96)


def test_tc_d128_aliased_p_stress_deterministic():
    # a long two-tile d = 128 run (P over S in TMEM, S_g(t+1) after P_g(t) V):
    # repeated runs bitwise identical and every row within 16-bit error of the
    # FP32 path — a read-after-write race on the aliased columns would show
    # as run-to-run differences or outliers
    g = torch.Generator(device=DEV)
    g.manual_seed(99)
    q, k, v = (torch.randn(1, 16, 8192, 128, device=DEV, generator=g) for _ in range(3))
    qb, kb, vb = q.bfloat16(), k.bfloat16(), v.bfloat16()
    y1 = elsa.scaled_dot_product_attention(qb, kb, vb)
    for _ in range(3):
        assert torch.equal(y1, elsa.scaled_dot_product_attention(qb, kb, vb))
    ref = elsa.scaled_dot_product_attention(qb.float(), kb.float(), vb.float())
    err = ((y1.float() - ref).norm(dim=-1) / ref.norm(dim=-1)).max().item()
    assert err < 2e-2, err


def test_tc_strided_out_and_expanded_kv():
    """A transposed `out` gets the values in the right elements (K5 writes a
    dense temporary, then copies); K/V expanded over heads (stride 0) are
    materialised instead of rejected."""
    g = torch.Generator(device=DEV)
    g.manual_seed(77)
    q = torch.randn(1, 4, 256, 64, device=DEV, generator=g).to(torch.bfloat16)
    k1 = torch.randn(1, 1, 300, 64, device=DEV, generator=g).to(torch.bfloat16)
    v1 = torch.randn(1, 1, 300, 64, device=DEV, generator=g).to(torch.bfloat16)
    k, v = k1.expand(1, 4, 300, 64), v1.expand(1, 4, 300, 64)
    assert k.stride(1) == 0
    ref = elsa.scaled_dot_product_attention(q, k.contiguous(), v.contiguous())
    y = elsa.scaled_dot_product_attention(q, k, v)
    assert torch.equal(y, ref)
    base = torch.empty(1, 4, 64, 256, device=DEV, dtype=torch.bfloat16)
    out = base.transpose(-1, -2)          # last-axis stride 256
    r = elsa.scaled_dot_product_attention(q, k, v, out=out)
    assert r.data_ptr() == out.data_ptr() and torch.equal(out, ref)


def test_requires_grad_is_rejected_loudly():
    q = torch.randn(1, 1, 64, 64, device=DEV, requires_grad=True)
    with pytest.raises(elsa.ShapeError):
        elsa.scaled_dot_product_attention(q, q.detach(), q.detach())
    with torch.no_grad():
        elsa.scaled_dot_product_attention(q, q, q)
