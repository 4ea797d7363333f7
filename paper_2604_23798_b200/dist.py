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
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import ShapeError

__all__ = ["chunk_bounds", "owned_chunks", "row_slices", "kv_sharded_attention",
           "shard_kv", "DEFAULT_CHUNKS"]

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


def kv_sharded_attention(q, k_local, v_local, kv_offset, n_kv, group=None,
                         chunks=DEFAULT_CHUNKS, gather=True, partial_fn=None, merge_fn=None):
    """Exact attention with keys sharded across the ranks of ``group``.

    ``q``: full (B, H, n_q, d) on this rank; ``k_local``/``v_local``: this
    rank's contiguous key rows starting at global key ``kv_offset`` (as
    returned by :func:`shard_kv`); ``n_kv``: total key count. Returns the full
    Y (B, H, n_q, dv) when ``gather`` else ``(row_begin, Y_rows)`` for this
    rank's row slice (rows ordered (b, h, q)).
    """
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
