"""Wide heads on the FP32 path: Q/K up to 256 floats (the w8r8d96 / w8r8d128 /
w4r8d256 kernels, raw Q staged in the K ring) and V of any width as 64-column slices (grid z),
through every entry that carries V columns — the forward (single launch and
kv splits + K2 merge), partial states, merge_states, the peer merge,
blockwise states + the block combine, and the host-buffer entry. The
reference accepts any head width (tensorio.py:83-112); the gate is the same
FP64 per-row bound as at d = 64 (verify.py:320-358)."""

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
U = 2.0 ** -24


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def _inputs(seed, b, h, n_q, n_kv, d, dv):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((b, h, n_q, d)).astype(np.float32)
    K = rng.standard_normal((b, h, n_kv, d)).astype(np.float32)
    V = rng.standard_normal((b, h, n_kv, dv)).astype(np.float32)
    return Q, K, V


def _bound(y, ref, n, what):
    err = oracle.row_rel_err(y, ref)
    thr = oracle.bound_threshold(n)
    assert err.max() <= thr, f"{what}: max row err {err.max():.3e} > {thr:.3e}"


@pytest.mark.parametrize("d,dv", [
    (128, 128), (128, 64), (64, 128), (96, 96), (80, 200), (65, 65), (127, 1), (100, 130),
    (128, 256), (16, 192), (128, 8), (96, 64), (88, 40), (72, 128), (256, 256), (192, 64),
    (200, 130), (129, 1), (256, 40), (32, 32), (17, 29), (32, 8), (4, 32), (96, 90), (70, 80),
    (96, 65), (64, 96), (128, 90), (100, 70), (200, 200), (192, 256), (256, 300)])
@pytest.mark.parametrize("splits", [1, 3])
def test_wide_heads_vs_fp64(d, dv, splits):
    n = 333
    Q, K, V = _inputs(d * 1000 + dv, 1, 2, n, n, d, dv)
    y = elsa.scaled_dot_product_attention(gpu(Q), gpu(K), gpu(V), kv_splits=splits,
                                          check_numerics=True)
    assert y.shape == (1, 2, n, dv)
    y = y.cpu().numpy()
    ref = oracle.naive_attention(Q, K, V)
    if dv <= 2:
        err = oracle.row_err_conditioned(y, Q, K, V, ref=ref)
        assert err.max() <= oracle.bound_threshold(n), err.max()
    else:
        _bound(y, ref, n, f"d{d} dv{dv} s{splits}")


def test_wide_heads_split_plan_is_bitwise_slice_consistent():
    # a slice's columns do not depend on how many other slices run: Y[..., :64]
    # of a dv = 192 problem equals the dv = 64 problem on V[..., :64] bitwise
    Q, K, V = _inputs(7, 2, 3, 700, 900, 128, 192)
    q, k, v = gpu(Q), gpu(K), gpu(V)
    for splits in (1, 4):
        y = elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits)
        for c in range(3):
            yc = elsa.scaled_dot_product_attention(q, k, v[..., 64 * c:64 * (c + 1)].contiguous(),
                                                   kv_splits=splits)
            assert torch.equal(y[..., 64 * c:64 * (c + 1)], yc)
        assert torch.equal(y, elsa.scaled_dot_product_attention(q, k, v, kv_splits=splits))


@pytest.mark.parametrize("n", [4096, 16384])
def test_wide_heads_large_sampled_rows(n):
    torch.manual_seed(n)
    q, k, v = (torch.randn(1, 2, n, 128, device=DEV) for _ in range(3))
    y = elsa.scaled_dot_product_attention(q, k, v, check_numerics=True)
    rng = np.random.default_rng(n)
    sc = 1.0 / math.sqrt(128)
    errs = []
    for h in range(2):
        K64, V64 = k[0, h].double().cpu().numpy(), v[0, h].double().cpu().numpy()
        for r in sorted(set([0, n - 1] + rng.integers(0, n, 48).tolist())):
            s = (K64 @ q[0, h, r].double().cpu().numpy()) * sc
            p = np.exp(s - s.max())
            ref = (p @ V64) / p.sum()
            got = y[0, h, r].double().cpu().numpy()
            errs.append(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert max(errs) <= oracle.bound_threshold(n), max(errs)


def test_wide_heads_strided_misaligned_and_negative_scale():
    rng = np.random.default_rng(11)
    n, d, dv = 150, 112, 100
    # row-strided views of wider buffers + a 4-byte-aligned base: generic loader
    qb = gpu(rng.standard_normal((1, 2, n, 128)).astype(np.float32))
    flat = gpu(rng.standard_normal(2 * n * d + 1).astype(np.float32))
    vb = gpu(rng.standard_normal((1, 2, n, 160)).astype(np.float32))
    q = qb[..., :d]
    k = flat[1:].view(1, 2, n, d)
    v = vb[..., 8:8 + dv]
    for scale in (None, -0.05, 0.0):
        y = elsa.scaled_dot_product_attention(q, k, v, scale=scale, check_numerics=True)
        ref = oracle.naive_attention(*(t.cpu().numpy() for t in (q, k, v)), scale=scale)
        _bound(y.cpu().numpy(), ref, n, f"scale={scale}")


def test_wide_partial_states_and_merge():
    n, d, dv = 500, 128, 150
    Q, K, V = _inputs(3, 1, 2, 260, n, d, dv)
    q, k, v = gpu(Q), gpu(K), gpu(V)
    for lo, hi, splits in ((0, 500, 1), (37, 300, 3), (0, 1, 1), (499, 500, 2)):
        m, S, W = (t.cpu().numpy() for t in elsa.partial_states(q, k, v, lo, hi, kv_splits=splits))
        m64, S64, W64 = oracle.partial_state_fp64(Q, K, V, lo, hi)
        np.testing.assert_allclose(m, m64, rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(S, S64 * np.exp(m64 - m.astype(np.float64)), rtol=1e-4)
        np.testing.assert_allclose(W / S[..., None], W64 / S64[..., None], rtol=1e-4, atol=1e-5)
    cuts = [0, 120, 120, 333, 500]
    parts = [elsa.partial_states(q, k, v, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    y = elsa.merge_states(*(torch.stack([p[i] for p in parts]) for i in range(3)))
    _bound(y.cpu().numpy(), oracle.naive_attention(Q, K, V), n, "merge")
    # non-finalized merge against the oracle's tree, every column slice
    mo, So, Wo = elsa.merge_states(*(torch.stack([p[i] for p in parts]) for i in range(3)),
                                   finalize=False)
    st = [tuple(t.cpu().numpy() for t in p) for p in parts]
    for r in (0, 77, 259):
        want = oracle.merge_tree([(s[0][0, 1, r], s[1][0, 1, r], s[2][0, 1, r]) for s in st])
        assert mo[0, 1, r].item() == want[0]
        np.testing.assert_allclose(Wo[0, 1, r].cpu().numpy(), want[2], rtol=4e-5, atol=4e-6)


def test_wide_peer_merge_matches_merge_states():
    n, dv = 300, 136
    Q, K, V = _inputs(5, 1, 1, 64, n, 96, dv)
    q, k, v = gpu(Q), gpu(K), gpu(V)
    cuts = [0, 80, 200, 300]
    parts = [elsa.partial_states(q, k, v, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    m, S, W = (torch.stack([p[i] for p in parts]).reshape(3, -1, *([dv] if i == 2 else []))
               .contiguous() for i in range(3))
    rows = m.shape[1]
    want = elsa.merge_states(m, S, W)
    # one "rank" holding all three chunks: the same pointers a 1-GPU run maps
    y = elsa.merge_peer_states([m.data_ptr()], [S.data_ptr()], [W.data_ptr()], 3, rows, 10,
                               rows - 10, dv)
    assert torch.equal(y, want[10:])


def test_wide_blockwise_states_and_combine():
    n, d, dv = 700, 128, 96
    Q, K, V = _inputs(9, 1, 2, 90, n, d, dv)
    q, k, v = gpu(Q), gpu(K), gpu(V)
    m, S, W = elsa.blockwise_states(q, k, v, block_size=128)
    assert W.shape == (1, 2, 90, 6, dv)
    m64, S64, W64 = oracle.blockwise_states_fp64(Q, K, V, 128)
    live = ~np.isneginf(m64)
    yb = (W.cpu().numpy() / S.cpu().numpy()[..., None])[live]
    yb64 = (W64 / S64[..., None])[live]
    err = np.linalg.norm(yb - yb64, axis=-1) / np.linalg.norm(yb64, axis=-1)
    assert err.max() <= U * oracle.scan_depth(128, 128) * 8, err.max()
    (tm, tS, tW), _ = elsa.inter_block_combine(m, S, W, return_prefixes=True)
    y = (tW / tS[..., None]).cpu().numpy()
    _bound(y, oracle.naive_attention(Q, K, V), n, "block combine")


def test_wide_host_entry_matches_device_bitwise():
    g = torch.Generator().manual_seed(1)
    q, k, v = (torch.randn(1, 6, 1000, w, generator=g).pin_memory() for w in (128, 128, 192))
    y_host = elsa.attention_from_host(q, k, v)
    y_dev = elsa.scaled_dot_product_attention(q.to(DEV), k.to(DEV), v.to(DEV))
    assert torch.equal(y_host, y_dev.cpu())


def test_too_wide_rejected():
    q = torch.randn(1, 1, 8, 257, device=DEV)
    v = torch.randn(1, 1, 8, 64, device=DEV)
    with pytest.raises(elsa.ShapeError):
        elsa.scaled_dot_product_attention(q, q, v)
    with pytest.raises(elsa.ShapeError):
        elsa.scaled_dot_product_attention(v, v, torch.randn(1, 1, 8, 4097, device=DEV))


_COPY_ENGINE_CHILD = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["ELSA_REPO"])
import paper_2604_23798_b200 as elsa
out = {}
for i, (n, d, dv) in enumerate(((300, 64, 64), (257, 96, 130), (200, 128, 128), (150, 256, 72))):
    g = torch.Generator().manual_seed(i)
    q, k, v = (torch.randn(1, 2, n, w, generator=g).cuda() for w in (d, d, dv))
    out[f"y{i}"] = elsa.scaled_dot_product_attention(q, k, v).cpu().numpy()
np.savez(sys.argv[1], **out)
"""


def test_copy_engine_bitwise_equals_tma(tmp_path):
    # the copy engine (forced for every operand) fills the same shared-memory
    # layouts as TMA, so Y must be bitwise identical to the TMA path's
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "ce.npz"
    env = dict(os.environ, ELSA_FORCE_GENERIC_LOAD="1", ELSA_REPO=repo)
    subprocess.run([sys.executable, "-c", _COPY_ENGINE_CHILD, str(out)], env=env, check=True,
                   timeout=300)
    ce = np.load(out)
    for i, (n, d, dv) in enumerate(((300, 64, 64), (257, 96, 130), (200, 128, 128), (150, 256, 72))):
        g = torch.Generator().manual_seed(i)
        q, k, v = (torch.randn(1, 2, n, w, generator=g).to(DEV) for w in (d, d, dv))
        y = elsa.scaled_dot_product_attention(q, k, v).cpu().numpy()
        assert np.array_equal(y, ce[f"y{i}"]), (n, d, dv)


@pytest.mark.parametrize("seed", range(24))
def test_random_geometry_fuzz(seed):
    # seeded random shapes / widths / views / splits / scales against FP64
    rng = np.random.default_rng(1000 + seed)
    B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
    n_q, n_kv = int(rng.integers(1, 400)), int(rng.integers(1, 700))
    d, dv = int(rng.integers(1, 257)), int(rng.integers(1, 300))
    pad = int(rng.integers(0, 3)) * 4            # row padding (keeps 16-byte rows when 0 or 4k)
    off = int(rng.integers(0, 2))                # 4-byte base offset -> copy engine
    splits = int(rng.choice([0, 1, 2, 5]))
    scale = None if rng.random() < 0.5 else float(rng.uniform(-0.3, 0.3))

    def make(n, w):
        base = torch.from_numpy(rng.standard_normal(B * H * n * (w + pad) + off)
                                .astype(np.float32)).to(DEV)
        return base[off:].view(B, H, n, w + pad)[..., :w]

    q, k, v = make(n_q, d), make(n_kv, d), make(n_kv, dv)
    y = elsa.scaled_dot_product_attention(q, k, v, scale=scale, kv_splits=splits,
                                          check_numerics=True).cpu().numpy()
    Q, K, V = (t.cpu().numpy() for t in (q, k, v))
    ref = oracle.naive_attention(Q, K, V, scale=scale)
    err = oracle.row_err_conditioned(y, Q, K, V, ref=ref, scale=scale)
    thr = oracle.bound_threshold(n_kv)
    assert err.max() <= thr, (B, H, n_q, n_kv, d, dv, pad, off, splits, scale, err.max())


@pytest.mark.parametrize("seed", range(12))
def test_random_partial_states_and_host_fuzz(seed):
    # partial states over random key ranges / split counts vs FP64, and the
    # host-buffer entry vs the device entry (bitwise) on random geometries
    rng = np.random.default_rng(5000 + seed)
    B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
    n_q, n_kv = int(rng.integers(1, 300)), int(rng.integers(2, 600))
    d, dv = int(rng.integers(1, 257)), int(rng.integers(1, 200))
    Q, K, V = _inputs(seed, B, H, n_q, n_kv, d, dv)
    q, k, v = gpu(Q), gpu(K), gpu(V)
    lo = int(rng.integers(0, n_kv - 1))
    hi = int(rng.integers(lo + 1, n_kv + 1))
    splits = int(rng.choice([0, 1, 2, 3, 8]))
    m, S, W = (t.cpu().numpy() for t in elsa.partial_states(q, k, v, lo, hi, kv_splits=splits))
    m64, S64, W64 = oracle.partial_state_fp64(Q, K, V, lo, hi)
    np.testing.assert_allclose(m, m64, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(S, S64 * np.exp(m64 - m.astype(np.float64)), rtol=2e-4)
    y = W / S[..., None]
    y64 = W64 / S64[..., None]
    mag = np.linalg.norm(np.abs(W64) / S64[..., None], axis=-1)
    err = np.linalg.norm(y - y64, axis=-1) / np.maximum(mag, 1e-300)
    assert err.max() <= oracle.bound_threshold(hi - lo), err.max()
    yh = elsa.attention_from_host(torch.from_numpy(Q), torch.from_numpy(K), torch.from_numpy(V))
    yd = elsa.scaled_dot_product_attention(q, k, v).cpu()
    assert torch.equal(yh, yd)


@pytest.mark.parametrize("seed", range(8))
def test_random_blockwise_fuzz(seed):
    # per-block states for random block sizes / widths, their combine, and the
    # exclusive prefixes, against FP64
    rng = np.random.default_rng(11000 + seed)
    B, H = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    n_q, n_kv = int(rng.integers(1, 120)), int(rng.integers(1, 700))
    d, dv = int(rng.integers(1, 257)), int(rng.integers(1, 160))
    bs = int(rng.choice([1, 7, 32, 64, 100, 128, 1000]))
    Q, K, V = _inputs(seed + 50, B, H, n_q, n_kv, d, dv)
    q, k, v = gpu(Q), gpu(K), gpu(V)
    m, S, W = elsa.blockwise_states(q, k, v, block_size=bs)
    nb = -(-n_kv // bs)
    assert W.shape == (B, H, n_q, nb, dv)
    m64, S64, W64 = oracle.blockwise_states_fp64(Q, K, V, bs)
    assert np.array_equal(np.isneginf(m.cpu().numpy()), np.isneginf(m64))
    (tm, tS, tW), (pm, pS, pW) = elsa.inter_block_combine(m, S, W, return_prefixes=True)
    y = (tW / tS[..., None]).cpu().numpy()
    ref = oracle.naive_attention(Q, K, V)
    err = oracle.row_err_conditioned(y, Q, K, V, ref=ref)
    assert err.max() <= oracle.bound_threshold(n_kv), err.max()
    assert torch.all(torch.isneginf(pm[..., 0])) and torch.all(pS[..., 0] == 0)
