"""The fused peer-memory exchange of the KV-sharded path on one GPU (world
size 1: the rank reads its own symmetric buffer through the same peer
pointers a multi-GPU run uses): bitwise equal to the NCCL all_to_all path and
within the FP64 bound."""

import os
import socket

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_2604_23798_b200 as elsa  # noqa: E402
from paper_2604_23798_b200 import dist as edist  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def pg():
    created = False
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(DEV)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
        created = True
    yield dist.group.WORLD
    if created:
        torch.cuda.synchronize()
        edist.release_peer_buffers()
        dist.destroy_process_group()


@pytest.mark.parametrize("B,H,n,chunks", [(1, 4, 1000, 8), (2, 3, 513, 4), (1, 2, 4096, 8)])
def test_peer_exchange_matches_nccl_and_oracle(pg, B, H, n, chunks):
    Q, K, V = oracle.generate(31, "regular", b=B, h=H, n=n, d=64, d_v=64, dtype=np.float32)
    q, k, v = (torch.from_numpy(x).to(DEV) for x in (Q, K, V))
    kl, vl, off = edist.shard_kv(k, v, 0, 1, chunks)
    y_nccl = edist.kv_sharded_attention(q, kl, vl, off, n, chunks=chunks, exchange="nccl")
    y_peer = edist.kv_sharded_attention(q, kl, vl, off, n, chunks=chunks, exchange="peer")
    y_again = edist.kv_sharded_attention(q, kl, vl, off, n, chunks=chunks, exchange="peer")
    elsa.check_device_error(DEV)
    assert torch.equal(y_nccl, y_peer) and torch.equal(y_peer, y_again)
    err = oracle.row_rel_err(y_peer.cpu().numpy(), oracle.naive_attention(Q, K, V))
    assert err.max() <= oracle.bound_threshold(n)
    lo, rows = edist.kv_sharded_attention(q, kl, vl, off, n, chunks=chunks, exchange="peer",
                                          gather=False)
    assert lo == 0 and torch.equal(rows, y_peer.reshape(-1, 64))


@pytest.mark.parametrize("B,H,n", [(1, 4, 1000), (2, 3, 513)])
def test_query_sharded_control_matches_direct(pg, B, H, n):
    g = torch.Generator(device=DEV)
    g.manual_seed(B * H + n)
    q, k, v = (torch.randn(B, H, n, 64, device=DEV, generator=g) for _ in range(3))
    y = edist.query_sharded_attention(q, k, v, gather=True)
    assert torch.equal(y, elsa.scaled_dot_product_attention(q, k, v))


@pytest.mark.parametrize("seed", range(6))
def test_kv_sharded_fuzz_widths_and_chunks(pg, seed):
    # random n_q != n_kv, head widths and chunk counts through both exchanges
    rng = np.random.default_rng(9000 + seed)
    B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
    n_q, n = int(rng.integers(1, 400)), int(rng.integers(8, 900))
    d, dv = int(rng.integers(1, 200)), int(rng.integers(1, 200))
    chunks = int(rng.choice([1, 2, 3, 5, 8]))
    Q = rng.standard_normal((B, H, n_q, d)).astype(np.float32)
    K = rng.standard_normal((B, H, n, d)).astype(np.float32)
    V = rng.standard_normal((B, H, n, dv)).astype(np.float32)
    q, k, v = (torch.from_numpy(x).to(DEV) for x in (Q, K, V))
    kl, vl, off = edist.shard_kv(k, v, 0, 1, chunks)
    y_nccl = edist.kv_sharded_attention(q, kl, vl, off, n, chunks=chunks, exchange="nccl")
    y_peer = edist.kv_sharded_attention(q, kl, vl, off, n, chunks=chunks, exchange="peer")
    elsa.check_device_error(DEV)
    assert torch.equal(y_nccl, y_peer)
    ref = oracle.naive_attention(Q, K, V)
    err = oracle.row_err_conditioned(y_peer.cpu().numpy(), Q, K, V, ref=ref)
    assert err.max() <= oracle.bound_threshold(n), err.max()


@pytest.mark.parametrize("ranks,per_rank,dv", [(2, 4, 64), (4, 2, 64), (8, 1, 64), (3, 2, 100),
                                               (16, 2, 8)])
def test_peer_merge_kernel_multi_rank_layout(ranks, per_rank, dv):
    # the fused merge as a multi-GPU run drives it, simulated on one GPU: each
    # "rank" owns per_rank consecutive chunks in its own buffer; every rank's
    # row slice merged through the peer kernel must equal merge_states over
    # all chunks in global order (rank-major, owned chunk minor), bitwise
    rng = np.random.default_rng(ranks * 10 + per_rank)
    chunks, rows = ranks * per_rank, 1000
    m = rng.uniform(-5, 5, (chunks, rows)).astype(np.float32)
    m[rng.random((chunks, rows)) < 0.05] = -np.inf
    S = rng.uniform(0.5, 4, (chunks, rows)).astype(np.float32)
    W = rng.standard_normal((chunks, rows, dv)).astype(np.float32)
    S[np.isneginf(m)] = 0
    W[np.isneginf(m)] = 0
    S[:, 7] = np.maximum(S[:, 7], 0.5)  # keep at least one live chunk per row
    m[0, :] = np.where(np.isneginf(m).all(axis=0), 0.0, m[0, :])
    S[0, :] = np.where(S.sum(axis=0) == 0, 1.0, S[0, :])
    mt, St, Wt = (torch.from_numpy(x).to(DEV) for x in (m, S, W))
    want = elsa.merge_states(mt, St, Wt)
    bufs = [(mt[r * per_rank:(r + 1) * per_rank].contiguous(),
             St[r * per_rank:(r + 1) * per_rank].contiguous(),
             Wt[r * per_rank:(r + 1) * per_rank].contiguous()) for r in range(ranks)]
    mp = [b[0].data_ptr() for b in bufs]
    Sp = [b[1].data_ptr() for b in bufs]
    Wp = [b[2].data_ptr() for b in bufs]
    for lo, hi in edist.row_slices(rows, ranks):
        y = elsa.merge_peer_states(mp, Sp, Wp, per_rank, rows, lo, hi - lo, dv)
        assert torch.equal(y, want[lo:hi]), (lo, hi)
