"""PyTorch-facing drop-in for the ELSA FP32 exact-attention path.

``scaled_dot_product_attention(q, k, v)`` replaces
``torch.nn.functional.scaled_dot_product_attention`` on ``(B, H, n, d)`` FP32
CUDA tensors (the entry point the paper describes, PAPER.md:18, :106-110,
:894-898) and runs the hand-written sm_100a kernels in ``libelsa.so``. It
mirrors the reference's computation ``scan_forward`` (engine.py:385-427):
exact softmax attention with scale ``1/sqrt(d)`` (tensorio.py:109-112),
strict FP32 arithmetic, deterministic output.

Non-goals of the reference are rejected loudly rather
than silently routed elsewhere: attention masks, causal masking, dropout,
non-FP32 dtypes and CPU tensors raise :class:`ShapeError`. There is no CPU or
PyTorch fallback anywhere on this path.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from .errors import NumericalError, ShapeError

__all__ = [
    "scaled_dot_product_attention",
    "attention_from_host",
    "partial_states",
    "merge_states",
    "merge_peer_states",
    "blockwise_states",
    "inter_block_combine",
    "check_device_error",
    "resolve_kv_splits",
    "describe_plan",
    "ffma_peak_tflops",
]



# Widest heads the FP32 kernels take (elsa_abi.cu kMaxD / kMaxDv): Q/K up to
# 256 floats wide; V of any width up to 4096 as column slices.
MAX_D = 256
MAX_DV = 4096

def _stream_ptr(device):
    idx = device.index if device.index is not None else torch.cuda.current_device()
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))


def _as_4d(t, name):
    if not isinstance(t, torch.Tensor):
        raise ShapeError(f"{name} must be a torch.Tensor")
    if t.dim() == 4:
        return t
    if t.dim() == 3:
        return t.unsqueeze(1)
    if t.dim() == 2:
        return t.unsqueeze(0).unsqueeze(0)
    if t.dim() > 4:
        # fold extra leading batch axes into B
        return t.reshape(-1, t.shape[-3], t.shape[-2], t.shape[-1])
    raise ShapeError(f"{name} must have at least 2 dimensions, got shape {tuple(t.shape)}")


_TC_DTYPES = (torch.float16, torch.bfloat16)
_SHAPE_CACHE = {}  # geometry -> (ElsaShape, workspace bytes) for the FP32 forward


def _validate(q, k, v, allow_16bit=False):
    for name, t in (("query", q), ("key", k), ("value", v)):
        if not isinstance(t, torch.Tensor):
            raise ShapeError(f"{name} must be a torch.Tensor")
        ok = t.dtype == torch.float32 or (allow_16bit and t.dtype in _TC_DTYPES)
        if not ok:
            raise ShapeError(
                f"{name} dtype {t.dtype}: the ELSA path takes torch.float32 (FP32 FFMA kernel)"
                + (" or float16 / bfloat16 (tcgen05 kernel)" if allow_16bit else "")
                + " only (no fallback)")
    if not (q.dtype == k.dtype == v.dtype):
        raise ShapeError("query, key and value must share one dtype")
    for name, t in (("query", q), ("key", k), ("value", v)):
        if not t.is_cuda:
            raise ShapeError(f"{name} is on {t.device}: libelsa runs on CUDA devices only "
                             "(no CPU fallback)")
    if not (q.device == k.device == v.device):
        raise ShapeError("query, key and value must be on the same device")


def _prep(t):
    # the ABI needs the last axis contiguous; other axes may be strided views
    if t.stride(-1) != 1 and t.shape[-1] > 1:
        t = t.contiguous()
    return t


def _shape(q, k, v, y=None):
    B, H, n_q, d = q.shape
    Bk, Hk, n_kv, dk = k.shape
    Bv, Hv, n_v, dv = v.shape
    if (Bk, Hk) != (B, H) or (Bv, Hv) != (B, H):
        raise ShapeError(f"batch/head dims differ: q {tuple(q.shape)}, k {tuple(k.shape)}, "
                         f"v {tuple(v.shape)}")
    if dk != d:
        raise ShapeError(f"key width {dk} != query width {d}")
    if n_v != n_kv:
        raise ShapeError(f"value length {n_v} != key length {n_kv}")
    if n_kv < 1:
        raise ShapeError("key/value length must be >= 1")
    if d > MAX_D or dv > MAX_DV:
        raise ShapeError(f"head dims d={d}, dv={dv}: libelsa supports d <= {MAX_D}, "
                         f"dv <= {MAX_DV}")
    s = _lib.ElsaShape()
    s.B, s.H, s.n_q, s.n_kv, s.d, s.dv = B, H, n_q, n_kv, d, dv
    for dst, t in ((s.q_stride, q), (s.k_stride, k), (s.v_stride, v)):
        dst[0], dst[1], dst[2] = t.stride(0), t.stride(1), t.stride(2)
    if y is not None:
        s.y_stride[0], s.y_stride[1], s.y_stride[2] = y.stride(0), y.stride(1), y.stride(2)
    return s


def check_device_error(device=None):
    """Synchronise the current stream and raise :class:`NumericalError` if a
    kernel flagged a zero / non-finite normalizer since the last check
    (engine.py:377-378)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    code = ctypes.c_int(0)
    with torch.cuda.device(dev):
        _lib.check_status(_lib.lib().elsa_get_device_error(_stream_ptr(dev), ctypes.byref(code)),
                          "elsa_get_device_error")
    if code.value == _lib.ELSA_ERR_NUMERICAL:
        raise NumericalError("softmax normalizer is zero or non-finite; inputs are corrupted")
    if code.value:
        _lib.check_status(code.value, "device")


def _plan_device(t):
    # planning only reads shapes and strides; host tensors plan for the current device
    return t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())


def resolve_kv_splits(q, k, v, kv_splits=0):
    """Split count elsa_fwd_f32 uses for these shapes (0 = auto)."""
    q4, k4, v4 = _as_4d(q, "query"), _as_4d(k, "key"), _as_4d(v, "value")
    shp = _shape(q4, k4, v4)
    with torch.cuda.device(_plan_device(q4)):
        r = _lib.lib().elsa_resolve_kv_splits(ctypes.byref(shp), int(kv_splits))
    if r < 0:
        _lib.check_status(-r, "elsa_resolve_kv_splits")
    return r


def workspace_bytes(q, k, v, kv_splits=0):
    """Split workspace elsa_fwd_f32 needs for these shapes (0 = none)."""
    q4, k4, v4 = _as_4d(q, "query"), _as_4d(k, "key"), _as_4d(v, "value")
    shp = _shape(q4, k4, v4)
    with torch.cuda.device(_plan_device(q4)):
        return int(_lib.lib().elsa_workspace_bytes(ctypes.byref(shp), int(kv_splits)))


def describe_plan(q, k, v, kv_splits=0):
    """The launch plan (kernel configuration, tiles, kv splits) for these shapes."""
    q4, k4, v4 = _as_4d(q, "query"), _as_4d(k, "key"), _as_4d(v, "value")
    shp = _shape(q4, k4, v4)
    buf = ctypes.create_string_buffer(256)
    with torch.cuda.device(_plan_device(q4)):
        _lib.check_status(_lib.lib().elsa_describe_plan(ctypes.byref(shp), int(kv_splits), buf, 256),
                          "elsa_describe_plan")
    return buf.value.decode()


def scaled_dot_product_attention(query, key, value, attn_mask=None, dropout_p=0.0,
                                 is_causal=False, scale=None, enable_gqa=False, *,
                                 kv_splits=0, check_numerics=False, out=None):
    """Exact FP32 softmax attention, drop-in for
    ``torch.nn.functional.scaled_dot_product_attention``.

    ``kv_splits`` (keyword-only) sets the number of contiguous key-range
    partitions merged by the fixed (+)-tree (0 = auto). ``check_numerics``
    synchronises and raises :class:`NumericalError` on a bad normalizer, the
    way the reference raises from ``scan_forward`` (engine.py:377-378).
    """
    if (enable_gqa and isinstance(query, torch.Tensor) and isinstance(key, torch.Tensor)
            and query.dim() >= 3 and key.dim() >= 3 and key.shape[-3] != query.shape[-3]):
        return _gqa_folded(query, key, value, attn_mask, dropout_p, is_causal, scale,
                           kv_splits, check_numerics, out)
    if (attn_mask is None and not dropout_p and not is_causal and out is None
            and not check_numerics):
        y = _fast_f32(query, key, value, scale, kv_splits)
        if y is not None:
            return y
    if attn_mask is not None:
        raise ShapeError("attn_mask is not supported: masks are a non-goal of the ELSA "
                         "FP32 path (SPEC.md:242)")
    if dropout_p:
        raise ShapeError("dropout is not supported on the exact-attention path")
    if is_causal:
        raise ShapeError("is_causal is not supported: the reference computes full "
                         "(bidirectional) attention only")
    _validate(query, key, value, allow_16bit=True)
    if torch.is_grad_enabled() and any(t.requires_grad for t in (query, key, value)):
        raise ShapeError("the ELSA path is forward-only (the reference has no backward): "
                         "call it under torch.no_grad() or on tensors without requires_grad "
                         "instead of silently cutting the gradient")
    orig_dim = query.dim()
    orig_shape = query.shape
    q, k, v = (_prep(_as_4d(t, n)) for t, n in ((query, "query"), (key, "key"), (value, "value")))
    d = q.shape[-1]
    sc = (1.0 / math.sqrt(d)) if scale is None else float(scale)
    if not math.isfinite(sc):
        raise ShapeError(f"scale must be finite, got {sc}")
    B, H, n_q, _ = q.shape
    dv = v.shape[-1]
    if q.dtype in _TC_DTYPES:
        y = _sdpa_tc(q, k, v, sc, out)
        if check_numerics:
            check_device_error(q.device)
        if orig_dim == 4 or out is not None:
            return y
        return y.reshape(*orig_shape[:-1], dv)
    if out is None:
        y = torch.empty((B, H, n_q, dv), device=q.device, dtype=torch.float32)
    else:
        y = out
        overlapping = any(s_ <= 0 for s_, n_ in zip(y.stride()[:3], y.shape[:3]) if n_ > 1)
        if tuple(y.shape) != (B, H, n_q, dv) or y.dtype != torch.float32 or y.device != q.device \
                or y.stride(-1) != 1 or overlapping:
            raise ShapeError("out must be a float32 (B, H, n_q, dv) tensor on the input device "
                             "with a contiguous last axis")
    # shape struct + workspace size per geometry (cheap repeat calls)
    key = (tuple(q.shape), q.stride(), tuple(k.shape), k.stride(), tuple(v.shape), v.stride(),
           y.stride(), int(kv_splits), q.device.index)
    hit = _SHAPE_CACHE.get(key)
    h = _lib.lib()
    with torch.cuda.device(q.device):
        if hit is None:
            shp = _shape(q, k, v, y)
            hit = (shp, h.elsa_workspace_bytes(ctypes.byref(shp), int(kv_splits)))
            if len(_SHAPE_CACHE) > 256:
                _SHAPE_CACHE.clear()
            _SHAPE_CACHE[key] = hit
        shp, ws_bytes = hit
        ws = (_split_workspace(q.device.index, torch._C._cuda_getCurrentRawStream(q.device.index),
                               ws_bytes) if ws_bytes else None)
        st = h.elsa_fwd_f32(
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.byref(shp),
            ctypes.c_double(sc), int(kv_splits),
            ctypes.c_void_p(ws.data_ptr() if ws is not None else 0), ctypes.c_size_t(ws_bytes),
            _stream_ptr(q.device))
        _lib.check_status(st, "elsa_fwd_f32")
        if check_numerics:
            check_device_error(q.device)
    if orig_dim == 4 or out is not None:
        return y
    return y.reshape(*orig_shape[:-1], dv)


def _gqa_folded(query, key, value, attn_mask, dropout_p, is_causal, scale, kv_splits,
                check_numerics, out):
    """Grouped-query attention (``enable_gqa``, H_q = g * H_kv; query head h
    reads key/value head h // g, torch's repeat_interleave semantics) without
    repeating K/V: the g query heads of one K/V head are folded into its query
    rows, (B, H_kv, g * n_q, d) — a view of a contiguous query — so one launch
    runs every group against its K/V once. Rows are independent, so the
    result is the same as with the heads expanded."""
    if value.dim() < 3 or value.shape[-3] != key.shape[-3]:
        raise ShapeError("key and value must have the same number of heads")
    # heads are dim -3 (torch's convention for enable_gqa); leading dims fold into B
    q4, k4, v4 = (t.reshape(-1, *t.shape[-3:]) for t in (query, key, value))
    if q4.shape[0] != k4.shape[0] or k4.shape[0] != v4.shape[0]:
        raise ShapeError(f"batch dims differ: q {tuple(query.shape)}, k {tuple(key.shape)}, "
                         f"v {tuple(value.shape)}")
    B, Hq, n_q, d = q4.shape
    Hk = k4.shape[1]
    if Hk < 1 or Hq % Hk:
        raise ShapeError(f"enable_gqa needs the query heads ({Hq}) to be a multiple of the "
                         f"key/value heads ({Hk})")
    g = Hq // Hk
    qf = q4.reshape(B, Hk, g * n_q, d)
    sc = (1.0 / math.sqrt(d)) if scale is None else scale
    y = scaled_dot_product_attention(qf, k4, v4, attn_mask, dropout_p, is_causal, sc, False,
                                     kv_splits=kv_splits, check_numerics=check_numerics)
    y = y.reshape(*query.shape[:-1], v4.shape[-1])
    if out is not None:
        if tuple(out.shape) != tuple(y.shape) or out.dtype != y.dtype or out.device != y.device:
            raise ShapeError("out must match the output's shape, dtype and device")
        out.copy_(y)
        return out
    return y


_FAST = {}   # (shapes, strides, kv_splits, device) -> (ElsaShape, ws bytes, scale, Y shape)
_SPLIT_WS = {}  # (device, stream) -> split workspace reused by calls on that stream


def _split_workspace(dev_idx, stream, nbytes):
    """Split workspace for elsa_fwd_f32, kept per (device, stream) and grown
    on demand: calls on one stream are ordered, so reuse is safe."""
    key = (dev_idx, stream)
    ws = _SPLIT_WS.get(key)
    if ws is None or ws.numel() < nbytes:
        if len(_SPLIT_WS) > 64:
            _SPLIT_WS.clear()
        ws = torch.empty(nbytes, device=torch.device("cuda", dev_idx), dtype=torch.uint8)
        _SPLIT_WS[key] = ws
    return ws


def _fast_f32(q, k, v, scale, kv_splits):
    """The common case without Python-side reshaping: 4-D float32 CUDA
    tensors on one device with contiguous last axes, no `out`, no gradient.
    Returns None to fall back to the general path (which validates and
    raises). Per-geometry state (the shape struct, workspace size, scale) is
    cached; the split workspace is reused per stream."""
    f32 = torch.float32
    if not (type(q) is torch.Tensor and type(k) is torch.Tensor and type(v) is torch.Tensor):
        return None
    if q.dtype is not f32 or k.dtype is not f32 or v.dtype is not f32:
        return None
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        return None
    if q.requires_grad or k.requires_grad or v.requires_grad:
        return None
    dev_idx = q.get_device()
    if dev_idx < 0 or k.get_device() != dev_idx or v.get_device() != dev_idx:
        return None
    qs, ks, vs = q.stride(), k.stride(), v.stride()
    if qs[3] != 1 or ks[3] != 1 or vs[3] != 1:
        return None
    key_ = (q.shape, qs, k.shape, ks, v.shape, vs, kv_splits, dev_idx, scale)
    hit = _FAST.get(key_)
    if hit is None:
        if any(x.shape[-1] == 0 for x in (q, k, v)):
            return None
        B, H, n_q, d = q.shape
        sc = (1.0 / math.sqrt(d)) if scale is None else float(scale)
        if not math.isfinite(sc):
            return None
        yshape = (B, H, n_q, v.shape[-1])
        shp = _shape(q, k, v)   # raises ShapeError on bad geometry
        dv = yshape[3]
        shp.y_stride[0], shp.y_stride[1], shp.y_stride[2] = H * n_q * dv, n_q * dv, dv
        with torch.cuda.device(q.device):
            ws_bytes = _lib.lib().elsa_workspace_bytes(ctypes.byref(shp), int(kv_splits))
        if len(_FAST) > 256:
            _FAST.clear()
        hit = (shp, ws_bytes, ctypes.c_double(sc), yshape)
        _FAST[key_] = hit
    shp, ws_bytes, sc, yshape = hit
    y = torch.empty(yshape, device=q.device, dtype=f32)
    stream = torch._C._cuda_getCurrentRawStream(dev_idx)
    ws_ptr = _split_workspace(dev_idx, stream, ws_bytes).data_ptr() if ws_bytes else 0
    h = _lib.lib()
    cur = torch._C._cuda_getDevice()
    if cur != dev_idx:
        torch._C._cuda_setDevice(dev_idx)
    try:
        st = h.elsa_fwd_f32(q.data_ptr(), k.data_ptr(), v.data_ptr(), y.data_ptr(),
                            ctypes.byref(shp), sc, int(kv_splits), ws_ptr, ws_bytes,
                            stream)
    finally:
        if cur != dev_idx:
            torch._C._cuda_setDevice(cur)
    if st:
        _lib.check_status(st, "elsa_fwd_f32")
    return y


_HOST_WS = {}


def _host_workspace(device, nbytes):
    """Device workspace of the host pipeline, kept per device and grown on
    demand (the library itself never allocates)."""
    ws = _HOST_WS.get(device.index)
    if ws is None or ws.numel() < nbytes:
        _HOST_WS.pop(device.index, None)
        ws = torch.empty(max(nbytes, 1), device=device, dtype=torch.uint8)
        _HOST_WS[device.index] = ws
    return ws


def _host_tensor(x, name):
    if isinstance(x, torch.Tensor):
        t = x
    else:
        import numpy as np
        t = torch.from_numpy(np.ascontiguousarray(x))
    if t.is_cuda:
        raise ShapeError(f"{name} is already on {t.device}: use scaled_dot_product_attention")
    if t.dtype != torch.float32:
        raise ShapeError(f"{name} dtype {t.dtype}: the host pipeline takes float32 only")
    return t.contiguous()


def attention_from_host(query, key, value, scale=None, *, out=None, kv_splits=0, device=None,
                        check_numerics=False, sync=True):
    """Exact FP32 attention on HOST (B, H, n, d) arrays computed on the GPU —
    the end-to-end form of the reference's ``scan_forward``, which takes and
    returns host arrays (engine.py:385-427).

    ``elsa_fwd_f32_host`` cuts the (b, h) heads into groups and overlaps each
    group's host->device copies, its forward kernels and its device->host copy
    on internal streams, ordered after prior work on the current stream.
    Page-locked inputs and ``out`` (``tensor.pin_memory()``) make the copies
    asynchronous. Returns ``out`` (a new CPU tensor if None); with ``sync``
    the call returns once Y is on the host, otherwise Y is complete when the
    current stream reaches this point."""
    q, k, v = (_host_tensor(t, n) for t, n in ((query, "query"), (key, "key"), (value, "value")))
    orig_shape = q.shape
    q, k, v = (_as_4d(t, n).contiguous() for t, n in ((q, "query"), (k, "key"), (v, "value")))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else \
        torch.device(device)
    d = q.shape[-1]
    sc = (1.0 / math.sqrt(d)) if scale is None else float(scale)
    if not math.isfinite(sc):
        raise ShapeError(f"scale must be finite, got {sc}")
    B, H, n_q, _ = q.shape
    dv = v.shape[-1]
    if out is None:
        # pageable: a fresh page-locked allocation per call would cost more than
        # the copy it speeds up (pass a pinned `out` to reuse one)
        y = torch.empty((B, H, n_q, dv), dtype=torch.float32)
    else:
        y = out
        if tuple(y.shape) != (B, H, n_q, dv) or y.dtype != torch.float32 or y.is_cuda \
                or not y.is_contiguous():
            raise ShapeError("out must be a contiguous float32 (B, H, n_q, dv) host tensor")
    shp = _shape(q, k, v, y)
    h = _lib.lib()
    with torch.cuda.device(dev):
        ws_bytes = h.elsa_host_workspace_bytes(ctypes.byref(shp), int(kv_splits))
        ws = _host_workspace(dev, ws_bytes)
        st = h.elsa_fwd_f32_host(
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.byref(shp),
            ctypes.c_double(sc), int(kv_splits), ctypes.c_void_p(ws.data_ptr()),
            ctypes.c_size_t(ws_bytes), _stream_ptr(dev))
        _lib.check_status(st, "elsa_fwd_f32_host")
        if check_numerics:
            check_device_error(dev)
        elif sync:
            torch.cuda.current_stream(dev).synchronize()
    if out is not None or len(orig_shape) == 4:
        return y
    return y.reshape(*orig_shape[:-1], dv)


def _sdpa_tc(q, k, v, sc, out):
    """FP16 / BF16 inputs: K5 on the tcgen05 tensor cores (FP32 accumulation
    and FP32 (m, S, W) state; output in the input format)."""
    B, H, n_q, d = q.shape
    dv = v.shape[-1]
    if d > 128 or dv > 128:
        raise ShapeError(f"the 16-bit tensor-core path takes d, dv <= 128, got d={d}, dv={dv}")

    def tma_ready(t):
        # TMA operands: 16-byte aligned base and row strides. Otherwise copy
        # into a buffer whose rows are padded to a multiple of 8 elements
        # (the kernel reads the first d columns; TMA zero-fills the box).
        # A zero stride (an expanded / broadcast axis, e.g. K/V shared across
        # heads) passes the modulo test but is no valid TMA stride:
        # materialise such inputs into the padded copy too.
        if t.stride(-1) == 1 and t.data_ptr() % 16 == 0 and all(
                s > 0 and (s * 2) % 16 == 0 for s, n in zip(t.stride()[:3], t.shape[:3])
                if n > 1):
            return t
        w = t.shape[-1]
        buf = torch.empty((*t.shape[:-1], -(-w // 8) * 8), device=t.device, dtype=t.dtype)
        buf[..., :w] = t
        return buf[..., :w]

    q, k, v = (tma_ready(t) for t in (q, k, v))
    dest = None
    if out is None:
        y = torch.empty((B, H, n_q, dv), device=q.device, dtype=q.dtype)
    else:
        y = out
        if tuple(y.shape) != (B, H, n_q, dv) or y.dtype != q.dtype or y.device != q.device:
            raise ShapeError("out must match the query's dtype/device with shape (B, H, n_q, dv)")
        if y.stride(-1) != 1 or any(s <= 0 for s, n in zip(y.stride()[:3], y.shape[:3])
                                    if n > 1):
            # K5 stores each Y row as contiguous columns: write a dense
            # temporary and copy it into the caller's strided view
            dest, y = y, torch.empty((B, H, n_q, dv), device=q.device, dtype=q.dtype)
    shp = _shape(q, k, v, y)
    with torch.cuda.device(q.device):
        st = _lib.lib().elsa_fwd_f16(
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.byref(shp),
            ctypes.c_double(sc), 1 if q.dtype == torch.bfloat16 else 0, _stream_ptr(q.device))
        _lib.check_status(st, "elsa_fwd_f16")
    if dest is not None:
        dest.copy_(y)
        return dest
    return y


def partial_states(query, key, value, kv_begin=0, kv_end=None, scale=None, kv_splits=1, *,
                   out=None):
    """The (m, S, W) summary of keys ``[kv_begin, kv_end)`` for every query —
    the per-chunk state of Proposition 1, as
    ``engine.blockwise_states`` + ``inter_block_combine`` produce on CPU
    (engine.py:430-451, 265-297). Returns ``m, S`` shaped (B, H, n_q) and
    ``W`` shaped (B, H, n_q, dv); ``m`` is in natural-log units, -inf for an
    empty range. ``out=(m, S, W)``: dense float32 CUDA tensors with
    B*H*n_q and B*H*n_q*dv elements to write into (e.g. views of a
    peer-mapped buffer)."""
    _validate(query, key, value)
    q, k, v = (_prep(_as_4d(t, n)) for t, n in ((query, "query"), (key, "key"), (value, "value")))
    B, H, n_q, d = q.shape
    n_kv, dv = k.shape[2], v.shape[-1]
    kv_end = n_kv if kv_end is None else int(kv_end)
    sc = (1.0 / math.sqrt(d)) if scale is None else float(scale)
    shp = _shape(q, k, v)
    if out is None:
        m = torch.empty((B, H, n_q), device=q.device, dtype=torch.float32)
        S = torch.empty_like(m)
        W = torch.empty((B, H, n_q, dv), device=q.device, dtype=torch.float32)
    else:
        m, S, W = out
        rows = B * H * n_q
        for name, t, numel in (("m", m, rows), ("S", S, rows), ("W", W, rows * dv)):
            if (t.dtype != torch.float32 or t.device != q.device or not t.is_contiguous()
                    or t.numel() != numel):
                raise ShapeError(f"out {name} must be a contiguous float32 tensor of {numel} "
                                 "elements on the input device")
    h = _lib.lib()
    with torch.cuda.device(q.device):
        # workspace for the internal split tree, sized for the requested count
        ws_bytes = 0
        if kv_splits != 1:
            # the plan (and its workspace) is made for the key range, not n_kv
            ws_bytes = h.elsa_partial_workspace_bytes(ctypes.byref(shp), int(kv_begin),
                                                      int(kv_end), int(kv_splits))
        ws = torch.empty(max(ws_bytes, 1), device=q.device, dtype=torch.uint8) if ws_bytes else None
        st = h.elsa_partial_f32(
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(v.data_ptr()), ctypes.byref(shp), ctypes.c_double(sc),
            int(kv_begin), int(kv_end), ctypes.c_void_p(m.data_ptr()),
            ctypes.c_void_p(S.data_ptr()), ctypes.c_void_p(W.data_ptr()), int(kv_splits),
            ctypes.c_void_p(ws.data_ptr() if ws is not None else 0), ctypes.c_size_t(ws_bytes),
            _stream_ptr(q.device))
        _lib.check_status(st, "elsa_partial_f32")
    return m, S, W


def merge_states(m, S, W, finalize=True):
    """Merge P partial states with the reference's balanced (+)-tree
    (monoid.py:234-265). ``m, S``: (P, *rows); ``W``: (P, *rows, dv), all FP32
    CUDA. ``finalize`` returns Y = W / S (*rows, dv); otherwise the merged
    ``(m, S, W)``."""
    for name, t in (("m", m), ("S", S), ("W", W)):
        if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda:
            raise ShapeError(f"{name} must be a float32 CUDA tensor")
    P = m.shape[0]
    rows_shape = tuple(m.shape[1:])
    dv = W.shape[-1]
    if tuple(S.shape) != tuple(m.shape) or tuple(W.shape[:-1]) != tuple(m.shape):
        raise ShapeError("m, S, W shapes disagree")
    rows = math.prod(rows_shape) if rows_shape else 1
    mc, Sc, Wc = m.contiguous(), S.contiguous(), W.contiguous()
    h = _lib.lib()
    with torch.cuda.device(m.device):
        if finalize:
            y = torch.empty((*rows_shape, dv), device=m.device, dtype=torch.float32)
            st = h.elsa_merge_f32(
                ctypes.c_void_p(mc.data_ptr()), ctypes.c_void_p(Sc.data_ptr()),
                ctypes.c_void_p(Wc.data_ptr()), int(P), int(rows), int(dv), int(rows), 1,
                ctypes.c_void_p(y.data_ptr()), None, None, None, _stream_ptr(m.device))
            _lib.check_status(st, "elsa_merge_f32")
            return y
        mo = torch.empty(rows_shape, device=m.device, dtype=torch.float32)
        So = torch.empty_like(mo)
        Wo = torch.empty((*rows_shape, dv), device=m.device, dtype=torch.float32)
        st = h.elsa_merge_f32(
            ctypes.c_void_p(mc.data_ptr()), ctypes.c_void_p(Sc.data_ptr()),
            ctypes.c_void_p(Wc.data_ptr()), int(P), int(rows), int(dv), int(rows), 0, None,
            ctypes.c_void_p(mo.data_ptr()), ctypes.c_void_p(So.data_ptr()),
            ctypes.c_void_p(Wo.data_ptr()), _stream_ptr(m.device))
        _lib.check_status(st, "elsa_merge_f32")
        return mo, So, Wo


def merge_peer_states(m_ptrs, S_ptrs, W_ptrs, per_rank, rows_total, row_lo, rows, dv, device=None):
    """Fused exchange + merge of the KV-sharded path (``elsa_merge_peers_f32``):
    rank r's state arrays live at the device pointers ``m_ptrs[r]``, ... (peer
    mapped, e.g. symmetric memory); returns Y for rows [row_lo, row_lo + rows)
    merged over all ranks' chunks in global chunk order."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    ranks = len(m_ptrs)
    arr = ctypes.c_void_p * ranks
    y = torch.empty((rows, dv), device=dev, dtype=torch.float32)
    with torch.cuda.device(dev):
        st = _lib.lib().elsa_merge_peers_f32(
            arr(*m_ptrs), arr(*S_ptrs), arr(*W_ptrs), int(ranks), int(per_rank),
            int(rows_total), int(row_lo), int(rows), int(dv), ctypes.c_void_p(y.data_ptr()),
            _stream_ptr(dev))
        _lib.check_status(st, "elsa_merge_peers_f32")
    return y


def blockwise_states(query, key, value, block_size=128, scale=None):
    """Per-key-block (m, S, W) states for every query row — the GPU form of
    ``engine.blockwise_states`` (engine.py:430-451), which returns the block
    totals of one query. Block j covers keys [j*B, min((j+1)*B, n_kv)).
    Returns ``m, S`` shaped (B, H, n_q, nblocks) and ``W`` shaped
    (B, H, n_q, nblocks, dv), natural-log anchors."""
    _validate(query, key, value)
    q, k, v = (_prep(_as_4d(t, n)) for t, n in ((query, "query"), (key, "key"), (value, "value")))
    B, H, n_q, d = q.shape
    n_kv, dv = k.shape[2], v.shape[-1]
    block_size = int(block_size)
    if block_size < 1:
        raise ShapeError(f"block size must be >= 1, got {block_size}")
    nb = -(-n_kv // block_size)
    sc = (1.0 / math.sqrt(d)) if scale is None else float(scale)
    shp = _shape(q, k, v)
    m = torch.empty((B, H, n_q, nb), device=q.device, dtype=torch.float32)
    S = torch.empty_like(m)
    W = torch.empty((B, H, n_q, nb, dv), device=q.device, dtype=torch.float32)
    with torch.cuda.device(q.device):
        st = _lib.lib().elsa_blockwise_f32(
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
            ctypes.c_void_p(v.data_ptr()), ctypes.byref(shp), ctypes.c_double(sc),
            int(block_size), ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(S.data_ptr()),
            ctypes.c_void_p(W.data_ptr()), _stream_ptr(q.device))
        _lib.check_status(st, "elsa_blockwise_f32")
    return m, S, W


def inter_block_combine(m, S, W, return_prefixes=False):
    """The reference's two-pass block combine on the GPU (engine.py:265-297):
    identity-padded up-sweep to each row's total and, with
    ``return_prefixes``, the down-sweep's exclusive per-block prefixes
    (identity first). ``m, S``: (*rows, K); ``W``: (*rows, K, dv), FP32 CUDA,
    natural-log anchors (the layout :func:`blockwise_states` returns)."""
    for name, t in (("m", m), ("S", S), ("W", W)):
        if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda:
            raise ShapeError(f"{name} must be a float32 CUDA tensor")
    if m.dim() < 1 or m.shape[-1] < 1:
        raise ShapeError("no block totals to combine")
    if tuple(S.shape) != tuple(m.shape) or tuple(W.shape[:-1]) != tuple(m.shape):
        raise ShapeError("m, S, W shapes disagree")
    K, dv = m.shape[-1], W.shape[-1]
    rows_shape = tuple(m.shape[:-1])
    rows = math.prod(rows_shape) if rows_shape else 1
    mc, Sc, Wc = m.contiguous(), S.contiguous(), W.contiguous()
    dev = m.device
    tm = torch.empty(rows_shape, device=dev, dtype=torch.float32)
    tS = torch.empty_like(tm)
    tW = torch.empty((*rows_shape, dv), device=dev, dtype=torch.float32)
    pre = None
    if return_prefixes:
        pre = (torch.empty_like(mc), torch.empty_like(Sc), torch.empty_like(Wc))
    h = _lib.lib()
    with torch.cuda.device(dev):
        ws_bytes = h.elsa_block_scan_workspace_bytes(int(rows), int(K), int(dv))
        if ws_bytes == 0 and rows > 0:
            raise ShapeError(f"unsupported block scan geometry (K={K}, dv={dv})")
        ws = torch.empty(max(ws_bytes, 1), device=dev, dtype=torch.uint8)
        ptr = (lambda t: ctypes.c_void_p(t.data_ptr()))
        st = h.elsa_block_scan_f32(
            ptr(mc), ptr(Sc), ptr(Wc), int(rows), int(K), int(dv), ptr(tm), ptr(tS), ptr(tW),
            *(ptr(t) for t in pre) if pre else (None, None, None),
            ptr(ws), ctypes.c_size_t(ws_bytes), _stream_ptr(dev))
        _lib.check_status(st, "elsa_block_scan_f32")
    return ((tm, tS, tW), pre) if return_prefixes else (tm, tS, tW)


def set_cluster_mode(mode):
    """Development aid: 0 = never merge kv splits inside the launch (always
    K1 + K2), 1 = when the planner's cost model prefers it (default), 2 =
    whenever the configuration allows it. Clears the per-geometry workspace
    cache, whose sizes depend on the mode."""
    h = _lib.lib()
    if not hasattr(h, "elsa_dev_set_cluster"):
        raise ShapeError("this libelsa build has no cluster-merge control")
    h.elsa_dev_set_cluster(int(mode))
    _SHAPE_CACHE.clear()
    _FAST.clear()


def set_tail_mode(mode):
    """Development aid: tail split of a one-split plan's last wave (0 = off,
    1 = the measured rule, s >= 2 = force s key pieces per tail unit)."""
    h = _lib.lib()
    if not hasattr(h, "elsa_dev_set_tail"):
        raise ShapeError("this libelsa build has no tail-split control")
    h.elsa_dev_set_tail(int(mode))
    _SHAPE_CACHE.clear()
    _FAST.clear()


def force_config(name=None):
    """Development aid: force one of the d <= 64 kernel configurations
    ("w4r8", "w8r8", "w8r16", or "w8r8acc", the two-level-accumulator kernel
    for long per-CTA chains); None restores the planner's choice."""
    h = _lib.lib()
    if not hasattr(h, "elsa_dev_force_config"):
        raise ShapeError("this libelsa build has no configuration control")
    h.elsa_dev_force_config(name.encode() if name else None)
    _SHAPE_CACHE.clear()
    _FAST.clear()


def ffma_peak_tflops(device=None):
    """Run the K4 FFMA microbenchmark on ``device`` and return TFLOP/s."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    out = ctypes.c_double(0.0)
    with torch.cuda.device(dev):
        _lib.check_status(_lib.lib().elsa_ffma_peak(_stream_ptr(dev), ctypes.byref(out)),
                          "elsa_ffma_peak")
    return out.value


def last_launch_count():
    """Kernels the last libelsa forward/partial/merge call launched on this thread."""
    return _lib.lib().elsa_last_launch_count()
