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
           "query_sharded_attention", "shard_kv", "DEFAULT_CHUNKS"]

DEFAULT_CHUNKS = 8


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


_PEER_BUFS = {}


def _peer_buffer(per, rows, dv, device, group):
    """Symmetric state buffer [m | S | W] for (per, rows, dv), rendezvoused once
    per shape and group and reused (the trailing barrier of every call keeps
    reuse safe)."""
    import torch.distributed._symmetric_memory as symm_mem

    key = (per, rows, dv, device.index, id(group))
    hit = _PEER_BUFS.get(key)
    if hit is None:
        n = per * rows * (2 + dv)
        buf = symm_mem.empty(n, dtype=torch.float32, device=device)
        grp = group if group is not None else dist.group.WORLD
        hdl = symm_mem.rendezvous(buf, grp)
        hit = (buf, hdl)
        _PEER_BUFS[key] = hit
    return hit


def _peer_exchange_merge(q, states_fn, per, rows, dv, chunks, group, rank, world):
    buf, hdl = _peer_buffer(per, rows, dv, q.device, group)
    m = buf[: per * rows].view(per, rows)
    S = buf[per * rows: 2 * per * rows].view(per, rows)
    W = buf[2 * per * rows:].view(per, rows, dv)
    states_fn(m, S, W)
    hdl.barrier(channel=0)  # every rank's states written (device-side, stream-ordered)
    lo, hi = row_slices(rows, world)[rank]
    base = [int(p) for p in hdl.buffer_ptrs]
    mp = [b for b in base]
    Sp = [b + per * rows * 4 for b in base]
    Wp = [b + 2 * per * rows * 4 for b in base]
    from .attention import merge_peer_states
    y_rows = merge_peer_states(mp, Sp, Wp, per, rows, lo, hi - lo, dv, device=q.device)
    hdl.barrier(channel=1)  # peers finished reading before the buffer is rewritten
    return lo, y_rows


def kv_sharded_attention(q, k_local, v_local, kv_offset, n_kv, group=None,
                         chunks=DEFAULT_CHUNKS, gather=True, partial_fn=None, merge_fn=None,
                         exchange="nccl"):
    """Exact attention with keys sharded across the ranks of ``group``.

    ``q``: full (B, H, n_q, d) on this rank; ``k_local``/``v_local``: this
    rank's contiguous key rows starting at global key ``kv_offset`` (as
    returned by :func:`shard_kv`); ``n_kv``: total key count. Returns the full
    Y (B, H, n_q, dv) when ``gather`` else ``(row_begin, Y_rows)`` for this
    rank's row slice (rows ordered (b, h, q)).
    """
    injected = partial_fn is not None or merge_fn is not None
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


def query_sharded_attention(q, k, v, group=None, gather=False):
    """The control experiment of SURVEY §8e: rank r computes the query rows of
    its slice (flattened (b, h, q) order, the same slices as the KV-sharded
    path) against ALL keys — no exchange, no merge. Returns ``(row_begin,
    Y_rows)``, or the full Y with ``gather``."""
    from .attention import scaled_dot_product_attention

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, H, n_q, d = q.shape
    dv = v.shape[-1]
    rows = B * H * n_q
    slices = row_slices(rows, world)
    lo, hi = slices[rank]
    # the slice = [partial head] + whole heads (one launch) + [partial head]
    qf, kf, vf = (t.reshape(B * H, 1, t.shape[2], t.shape[3]) for t in (q, k, v))
    out = torch.empty((hi - lo, dv), device=q.device, dtype=torch.float32)
    r = lo
    while r < hi:
        bh, q0 = divmod(r, n_q)
        if q0 == 0 and hi - r >= n_q:  # a run of whole heads
            nh = (hi - r) // n_q
            y = scaled_dot_product_attention(qf[bh:bh + nh].transpose(0, 1),
                                             kf[bh:bh + nh].transpose(0, 1),
                                             vf[bh:bh + nh].transpose(0, 1))
            out[r - lo: r - lo + nh * n_q] = y.reshape(nh * n_q, dv)
            r += nh * n_q
        else:
            q1 = min(n_q, q0 + (hi - r))
            y = scaled_dot_product_attention(qf[bh:bh + 1, :, q0:q1], kf[bh:bh + 1], vf[bh:bh + 1])
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
