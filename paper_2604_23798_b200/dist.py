"""KV-sharded multi-GPU ELSA attention: one process per GPU, NCCL exchange of
per-chunk (m, S, W) states, fixed (+)-tree merge on the owning rank.

Why this is exact: by Proposition 1 attention over the
full key range equals the (+)-combination, in key order, of the states of any
contiguous partition of the keys. The reference exposes exactly this
per-chunk contract on CPU (engine.blockwise_states + inter_block_combine,
engine.py:430-451 / 265-297; monoid.merge_tree, monoid.py:234-265).

Schedule (G ranks, C global key chunks, C a multiple of G; rank r holds all
of Q and the K/V rows of chunks [r*C/G, (r+1)*C/G)):

  1. each rank computes the (m, S, W) state of each owned chunk for every
     query row (``elsa_partial_f32`` — no inter-rank traffic);
  2. the query rows R = B*H*n_q are cut into G contiguous slices; one
     ``all_to_all_single`` sends slice j of every owned chunk state to rank j
     (per rank: (C/G)*R*(2+dv)*4 bytes out, the same in);
  3. rank j merges the C chunk states of its row slice with the balanced
     (+)-tree in global chunk order (``elsa_merge_f32``) and writes Y rows;
  4. optionally ``all_gather`` the Y slices.

Because C is fixed independently of G and each chunk's state is computed by
the same kernel over the same key range, the result is bitwise identical for
G = 1, 2, 4, 8 (the merge tree has the same C leaves in the same order).

The compute and merge steps are injectable (``partial_fn``, ``merge_fn``) so
the host logic — chunk plan, packing, exchange, tree order — is covered by
world-size-2 ``gloo`` tests on CPU; the product path uses libelsa kernels.

``exchange="peer"`` replaces steps 2-3 with one kernel: each rank writes its
chunk states into a symmetric (peer-mapped, NVLink) buffer
(``torch.distributed._symmetric_memory``), a device-side barrier orders the
ranks, and ``elsa_merge_peers_f32`` reads every rank's states for its row
slice straight from peer memory and merges them in registers — no
all_to_all, no staging copy, bitwise identical to the NCCL exchange.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import ShapeError

__all__ = ["chunk_bounds", "owned_chunks", "row_slices", "kv_sharded_attention",
           "query_sharded_attention", "shard_kv", "release_peer_buffers", "last_launch_count",
           "resolve_exchange",
           "DEFAULT_CHUNKS"]

DEFAULT_CHUNKS = 8


_LAUNCHES = [0]


def _tally():
    """Add the kernels the last libelsa call launched to this call's count."""
    from .attention import last_launch_count
    _LAUNCHES[0] += last_launch_count()


def last_launch_count():
    """Kernels the last kv_sharded_attention / query_sharded_attention call
    launched on this rank (libelsa kernels only; NCCL's are not counted)."""
    return _LAUNCHES[0]


def chunk_bounds(n_kv, chunks):
    """Global chunk c covers keys [c*n//C, (c+1)*n//C)."""
    if chunks < 1:
        raise ShapeError("chunks must be >= 1")
    return [(c * n_kv // chunks, (c + 1) * n_kv // chunks) for c in range(chunks)]


def owned_chunks(rank, world, chunks):
    if chunks % world:
        raise ShapeError(f"chunk count {chunks} must be a multiple of the world size {world}")
    per = chunks // world
    return list(range(rank * per, (rank + 1) * per))


def row_slices(rows, world):
    return [(j * rows // world, (j + 1) * rows // world) for j in range(world)]


def shard_kv(k, v, rank, world, chunks=DEFAULT_CHUNKS):
    """The K/V rows rank ``rank`` holds: keys of its owned chunks (contiguous)."""
    n_kv = k.shape[2]
    bounds = chunk_bounds(n_kv, chunks)
    own = owned_chunks(rank, world, chunks)
    lo, hi = bounds[own[0]][0], bounds[own[-1]][1]
    return k[:, :, lo:hi], v[:, :, lo:hi], lo


def _gpu_partial(q, k, v, kv_begin, kv_end):
    # auto splits: the planner caps the per-CTA key chain (accuracy at long
    # chunks); the plan depends only on the chunk's shape, so every world size
    # computes each global chunk identically
    from .attention import partial_states
    return partial_states(q, k, v, kv_begin, kv_end, kv_splits=0)


def _gpu_merge(m, S, W):
    from .attention import merge_states
    return merge_states(m, S, W, finalize=True)


# One symmetric state buffer per (device, group), grown on demand and reused
# as a prefix for smaller shapes, so varying sequence lengths do not pile up
# peer-mapped allocations (release_peer_buffers() frees them).
_PEER_BUFS = {}


def release_peer_buffers():
    """Drop the cached symmetric-memory state buffers (call on every rank)."""
    _PEER_BUFS.clear()


def _peer_buffer(per, rows, dv, device, group):
    """Symmetric state buffer holding at least per*rows*(2+dv) floats,
    rendezvoused on first use (and when a larger shape needs a bigger one) and
    reused; the trailing barrier of every call keeps reuse safe. Every rank
    runs the same shape sequence, so the collective rendezvous stays matched."""
    import os
    # only unicast peer pointers (buffer_ptrs) are read; the NVLS multicast
    # object symmetric memory would also try to export is not needed
    os.environ.setdefault("TORCH_SYMM_MEM_DISABLE_MULTICAST", "1")
    import torch.distributed._symmetric_memory as symm_mem

    key = (device.index, id(group))
    need = per * rows * (2 + dv)
    hit = _PEER_BUFS.get(key)
    if hit is None or hit[0].numel() < need:
        _PEER_BUFS.pop(key, None)
        buf = symm_mem.empty(need, dtype=torch.float32, device=device)
        grp = group if group is not None else dist.group.WORLD
        hdl = symm_mem.rendezvous(buf, grp)
        hit = (buf, hdl)
        _PEER_BUFS[key] = hit
    return hit


def _peer_exchange_merge(q, states_fn, per, rows, dv, chunks, group, rank, world):
    buf, hdl = _peer_buffer(per, rows, dv, q.device, group)
    m = buf[: per * rows].view(per, rows)
    S = buf[per * rows: 2 * per * rows].view(per, rows)
    W = buf[2 * per * rows: per * rows * (2 + dv)].view(per, rows, dv)
    states_fn(m, S, W)
    hdl.barrier(channel=0)  # every rank's states written (device-side, stream-ordered)
    lo, hi = row_slices(rows, world)[rank]
    base = [int(p) for p in hdl.buffer_ptrs]
    mp = [b for b in base]
    Sp = [b + per * rows * 4 for b in base]
    Wp = [b + 2 * per * rows * 4 for b in base]
    from .attention import merge_peer_states
    y_rows = merge_peer_states(mp, Sp, Wp, per, rows, lo, hi - lo, dv, device=q.device)
    _tally()
    hdl.barrier(channel=1)  # peers finished reading before the buffer is rewritten
    return lo, y_rows


def resolve_exchange(exchange, q, group=None, injected=False):
    """``"auto"`` -> ``"peer"`` when the group runs NCCL on CUDA tensors and
    the libelsa kernels do the compute, else ``"nccl"`` (the packed
    all_to_all path, which also serves gloo / CPU and world size 1)."""
    if exchange != "auto":
        return exchange
    use_peer = (not injected and q.is_cuda and dist.is_initialized()
                and dist.get_backend(group) == "nccl")
    return "peer" if use_peer else "nccl"


def kv_sharded_attention(q, k_local, v_local, kv_offset, n_kv, group=None,
                         chunks=DEFAULT_CHUNKS, gather=True, partial_fn=None, merge_fn=None,
                         exchange="auto"):
    """Exact attention with keys sharded across the ranks of ``group``.

    ``q``: full (B, H, n_q, d) on this rank; ``k_local``/``v_local``: this
    rank's contiguous key rows starting at global key ``kv_offset`` (as
    returned by :func:`shard_kv`); ``n_kv``: total key count. Returns the full
    Y (B, H, n_q, dv) when ``gather`` else ``(row_begin, Y_rows)`` for this
    rank's row slice (rows ordered (b, h, q)).

    ``exchange``: ``"peer"`` (the fused symmetric-memory merge), ``"nccl"``
    (all_to_all + K2) or ``"auto"`` (default): peer when the process group
    runs the NCCL backend on CUDA tensors and no compute step is injected,
    else nccl (which at world size 1 needs no process group at all).
    """
    injected = partial_fn is not None or merge_fn is not None
    _LAUNCHES[0] = 0
    partial_fn = partial_fn or _gpu_partial
    merge_fn = merge_fn or _gpu_merge
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, H, n_q, _ = q.shape
    dv = v_local.shape[-1]
    rows = B * H * n_q
    bounds = chunk_bounds(n_kv, chunks)
    own = owned_chunks(rank, world, chunks)
    per = len(own)
    if kv_offset != bounds[own[0]][0] or kv_offset + k_local.shape[2] != bounds[own[-1]][1]:
        raise ShapeError("local K/V rows do not match this rank's chunk range")

    exchange = resolve_exchange(exchange, q, group, injected)
    if exchange == "peer":
        if injected:
            raise ShapeError("the peer exchange runs the libelsa kernels only")
        if chunks > 32 or world > 16:
            raise ShapeError("the peer merge handles <= 32 chunks over <= 16 ranks")

        def states_fn(m, S, W):
            from .attention import partial_states
            for i, c in enumerate(own):
                lo, hi = bounds[c]
                partial_states(q, k_local, v_local, lo - kv_offset, hi - kv_offset, kv_splits=0,
                               out=(m[i], S[i], W[i]))
                _tally()

        my_lo, y_rows = _peer_exchange_merge(q, states_fn, per, rows, dv, chunks, group, rank,
                                             world)
        if not gather:
            return my_lo, y_rows
        slices = row_slices(rows, world)
        if world == 1:
            return y_rows.reshape(B, H, n_q, dv)
        maxr = max(hi - lo for lo, hi in slices)
        pad = torch.zeros((maxr, dv), dtype=torch.float32, device=q.device)
        pad[: y_rows.shape[0]] = y_rows
        outs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        y = torch.cat([o[: hi - lo] for o, (lo, hi) in zip(outs, slices)])
        return y.reshape(B, H, n_q, dv)
    if exchange != "nccl":
        raise ShapeError(f"exchange must be 'nccl' or 'peer', got {exchange!r}")

    # 1. per-chunk states, packed [chunk][row][2 + dv]
    states = torch.empty((per, rows, 2 + dv), dtype=torch.float32, device=q.device)
    for i, c in enumerate(own):
        lo, hi = bounds[c]
        m, S, W = partial_fn(q, k_local, v_local, lo - kv_offset, hi - kv_offset)
        if not injected:
            _tally()
        states[i, :, 0] = m.reshape(rows)
        states[i, :, 1] = S.reshape(rows)
        states[i, :, 2:] = W.reshape(rows, dv)

    slices = row_slices(rows, world)
    my_lo, my_hi = slices[rank]
    my_rows = my_hi - my_lo
    if world == 1:
        gathered = states.unsqueeze(0)  # [src=1][chunk][rows][2+dv]
    else:
        # 2. send row slice j of every owned chunk to rank j
        send = torch.cat([states[:, lo:hi].reshape(-1) for lo, hi in slices])
        in_sizes = [per * (hi - lo) * (2 + dv) for lo, hi in slices]
        out_sizes = [per * my_rows * (2 + dv)] * world
        recv = torch.empty(sum(out_sizes), dtype=torch.float32, device=q.device)
        dist.all_to_all_single(recv, send, output_split_sizes=out_sizes,
                               input_split_sizes=in_sizes, group=group)
        gathered = recv.view(world, per, my_rows, 2 + dv)
    # global chunk order: source rank major, owned chunk minor
    allc = gathered.reshape(chunks, my_rows, 2 + dv)
    # 3. fixed balanced tree over the C chunk states
    y_rows = merge_fn(allc[..., 0].contiguous(), allc[..., 1].contiguous(),
                      allc[..., 2:].contiguous())
    if not injected:
        _tally()
    if not gather:
        return my_lo, y_rows
    if world == 1:
        return y_rows.reshape(B, H, n_q, dv)
    # 4. all-gather the row slices (uneven sizes: pad to the largest slice)
    maxr = max(hi - lo for lo, hi in slices)
    pad = torch.zeros((maxr, dv), dtype=torch.float32, device=q.device)
    pad[:my_rows] = y_rows
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    y = torch.cat([o[: hi - lo] for o, (lo, hi) in zip(outs, slices)])
    return y.reshape(B, H, n_q, dv)


def query_sharded_attention(q, k, v, group=None, gather=False, attn_fn=None):
    """Batch x heads sharding (BASELINE north_star; SURVEY §8e's control
    experiment): rank r computes the query rows of its slice (flattened
    (b, h, q) order, the same slices as the KV-sharded path) against ALL keys
    — no exchange, no merge. A slice that starts or ends inside a head runs
    that head's partial query range; the whole heads between run as one
    launch. Returns ``(row_begin, Y_rows)``, or the full Y with ``gather``.
    ``attn_fn(q, k, v) -> y`` (default: the libelsa forward) is injectable so
    the slicing is testable on CPU."""
    injected = attn_fn is not None
    if attn_fn is None:
        from .attention import scaled_dot_product_attention as attn_fn

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, H, n_q, d = q.shape
    dv = v.shape[-1]
    rows = B * H * n_q
    slices = row_slices(rows, world)
    lo, hi = slices[rank]
    _LAUNCHES[0] = 0
    # the slice = [partial head] + whole heads (one launch) + [partial head];
    # heads as one (1, B*H, n, d) batch (a view for contiguous inputs), whole
    # heads written straight into the output rows (no staging copy)
    qf, kf, vf = (t.reshape(1, B * H, t.shape[2], t.shape[3]) for t in (q, k, v))
    out = torch.empty((hi - lo, dv), device=q.device, dtype=torch.float32)
    r = lo
    while r < hi:
        bh, q0 = divmod(r, n_q)
        if q0 == 0 and hi - r >= n_q:  # a run of whole heads
            nh = (hi - r) // n_q
            dst = out[r - lo: r - lo + nh * n_q].view(1, nh, n_q, dv)
            if injected:
                dst.copy_(attn_fn(qf[:, bh:bh + nh], kf[:, bh:bh + nh], vf[:, bh:bh + nh])
                          .reshape(1, nh, n_q, dv))
            else:
                attn_fn(qf[:, bh:bh + nh], kf[:, bh:bh + nh], vf[:, bh:bh + nh], out=dst)
                _tally()
            r += nh * n_q
        else:
            q1 = min(n_q, q0 + (hi - r))
            y = attn_fn(qf[:, bh:bh + 1, q0:q1], kf[:, bh:bh + 1], vf[:, bh:bh + 1])
            if not injected:
                _tally()
            out[r - lo: r - lo + (q1 - q0)] = y.reshape(q1 - q0, dv)
            r += q1 - q0
    if not gather:
        return lo, out
    if world == 1:
        return out.reshape(B, H, n_q, dv)
    maxr = max(b_ - a_ for a_, b_ in slices)
    pad = torch.zeros((maxr, dv), dtype=torch.float32, device=q.device)
    pad[: out.shape[0]] = out
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    y = torch.cat([o[: b_ - a_] for o, (a_, b_) in zip(outs, slices)])
    return y.reshape(B, H, n_q, dv)
