"""ctypes binding of ``libelsa.so`` (the C-ABI in ``include/elsa.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2604_23798_b200``) and loaded from this package directory.
There is no fallback: if the library is missing or fails to load, every
compute entry point raises :class:`ElsaLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ElsaCudaError, ElsaLibraryError, NumericalError, ShapeError, WorkspaceError

__all__ = ["lib", "ElsaShape", "check_status", "LIB_PATH", "EXPORTED_SYMBOLS"]

LIB_PATH = os.environ.get("ELSA_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libelsa.so")  # env override: build A/B experiments

# Every symbol include/elsa.h declares.
EXPORTED_SYMBOLS = (
    "elsa_abi_version",
    "elsa_strerror",
    "elsa_scan_depth",
    "elsa_resolve_kv_splits",
    "elsa_workspace_bytes",
    "elsa_partial_workspace_bytes",
    "elsa_fwd_f32",
    "elsa_host_workspace_bytes",
    "elsa_fwd_f32_host",
    "elsa_partial_f32",
    "elsa_fwd_f16",
    "elsa_merge_f32",
    "elsa_merge_peers_f32",
    "elsa_blockwise_f32",
    "elsa_block_scan_workspace_bytes",
    "elsa_block_scan_f32",
    "elsa_device_alloc",
    "elsa_device_free",
    "elsa_get_device_error",
    "elsa_ffma_peak",
    "elsa_last_launch_count",
    "elsa_last_cuda_error",
    "elsa_describe_plan",
)

ABI_VERSION = 1

ELSA_OK = 0
ELSA_ERR_SHAPE = 2
ELSA_ERR_NUMERICAL = 3
ELSA_ERR_CUDA = 5
ELSA_ERR_NCCL = 6
ELSA_ERR_WORKSPACE = 7


class ElsaShape(ctypes.Structure):
    """Mirror of ``elsa_shape`` (include/elsa.h)."""

    _fields_ = [
        ("B", ctypes.c_int64),
        ("H", ctypes.c_int64),
        ("n_q", ctypes.c_int64),
        ("n_kv", ctypes.c_int64),
        ("d", ctypes.c_int64),
        ("dv", ctypes.c_int64),
        ("q_stride", ctypes.c_int64 * 3),
        ("k_stride", ctypes.c_int64 * 3),
        ("v_stride", ctypes.c_int64 * 3),
        ("y_stride", ctypes.c_int64 * 3),
    ]


_lock = threading.Lock()
_lib = None


def _declare(h):
    c_int, c_i64, c_sz, c_vp, c_dbl = (ctypes.c_int, ctypes.c_int64, ctypes.c_size_t,
                                       ctypes.c_void_p, ctypes.c_double)
    shp = ctypes.POINTER(ElsaShape)
    h.elsa_abi_version.restype = c_int
    h.elsa_abi_version.argtypes = []
    h.elsa_strerror.restype = ctypes.c_char_p
    h.elsa_strerror.argtypes = [c_int]
    h.elsa_scan_depth.restype = c_int
    h.elsa_scan_depth.argtypes = [c_i64, c_i64]
    h.elsa_resolve_kv_splits.restype = c_int
    h.elsa_resolve_kv_splits.argtypes = [shp, c_int]
    h.elsa_workspace_bytes.restype = c_sz
    h.elsa_workspace_bytes.argtypes = [shp, c_int]
    h.elsa_partial_workspace_bytes.restype = c_sz
    h.elsa_partial_workspace_bytes.argtypes = [shp, c_i64, c_i64, c_int]
    # development aid (not in include/elsa.h): cluster-merge mode 0 / 1 / 2
    if hasattr(h, "elsa_dev_set_cluster"):
        h.elsa_dev_set_cluster.restype = None
        h.elsa_dev_set_cluster.argtypes = [c_int]
    if hasattr(h, "elsa_dev_set_tail"):
        h.elsa_dev_set_tail.restype = None
        h.elsa_dev_set_tail.argtypes = [c_int]
    if hasattr(h, "elsa_dev_force_config"):
        h.elsa_dev_force_config.restype = None
        h.elsa_dev_force_config.argtypes = [ctypes.c_char_p]
    h.elsa_fwd_f32.restype = c_int
    h.elsa_fwd_f32.argtypes = [c_vp, c_vp, c_vp, c_vp, shp, c_dbl, c_int, c_vp, c_sz, c_vp]
    h.elsa_host_workspace_bytes.restype = c_sz
    h.elsa_host_workspace_bytes.argtypes = [shp, c_int]
    h.elsa_fwd_f32_host.restype = c_int
    h.elsa_fwd_f32_host.argtypes = [c_vp, c_vp, c_vp, c_vp, shp, c_dbl, c_int, c_vp, c_sz, c_vp]
    h.elsa_partial_f32.restype = c_int
    h.elsa_partial_f32.argtypes = [c_vp, c_vp, c_vp, shp, c_dbl, c_i64, c_i64,
                                   c_vp, c_vp, c_vp, c_int, c_vp, c_sz, c_vp]
    h.elsa_fwd_f16.restype = c_int
    h.elsa_fwd_f16.argtypes = [c_vp, c_vp, c_vp, c_vp, shp, c_dbl, c_int, c_vp]
    h.elsa_merge_f32.restype = c_int
    h.elsa_merge_f32.argtypes = [c_vp, c_vp, c_vp, c_int, c_i64, c_int, c_i64, c_int,
                                 c_vp, c_vp, c_vp, c_vp, c_vp]
    h.elsa_merge_peers_f32.restype = c_int
    h.elsa_merge_peers_f32.argtypes = [ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                       ctypes.POINTER(c_vp), c_int, c_int, c_i64, c_i64, c_i64,
                                       c_int, c_vp, c_vp]
    h.elsa_blockwise_f32.restype = c_int
    h.elsa_blockwise_f32.argtypes = [c_vp, c_vp, c_vp, shp, c_dbl, c_i64, c_vp, c_vp, c_vp, c_vp]
    h.elsa_block_scan_workspace_bytes.restype = c_sz
    h.elsa_block_scan_workspace_bytes.argtypes = [c_i64, c_int, c_int]
    h.elsa_block_scan_f32.restype = c_int
    h.elsa_block_scan_f32.argtypes = [c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]
    h.elsa_device_alloc.restype = c_int
    h.elsa_device_alloc.argtypes = [c_sz, ctypes.POINTER(c_vp)]
    h.elsa_device_free.restype = c_int
    h.elsa_device_free.argtypes = [c_vp]
    h.elsa_get_device_error.restype = c_int
    h.elsa_get_device_error.argtypes = [c_vp, ctypes.POINTER(c_int)]
    h.elsa_ffma_peak.restype = c_int
    h.elsa_ffma_peak.argtypes = [c_vp, ctypes.POINTER(c_dbl)]
    h.elsa_last_launch_count.restype = c_int
    h.elsa_last_launch_count.argtypes = []
    h.elsa_last_cuda_error.restype = ctypes.c_char_p
    h.elsa_last_cuda_error.argtypes = []
    h.elsa_describe_plan.restype = c_int
    h.elsa_describe_plan.argtypes = [shp, c_int, ctypes.c_char_p, c_sz]


def lib():
    """Load (once) and return the ctypes handle to ``libelsa.so``."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ElsaLibraryError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (no CPU fallback exists)")
            try:
                h = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise ElsaLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(h)
            if h.elsa_abi_version() != ABI_VERSION:
                raise ElsaLibraryError(
                    f"libelsa ABI {h.elsa_abi_version()} != expected {ABI_VERSION}")
            _lib = h
    return _lib


def strerror(status):
    return lib().elsa_strerror(int(status)).decode()


def check_status(status, what="elsa"):
    """Raise the reference-taxonomy exception for a non-zero status."""
    if status == ELSA_OK:
        return
    msg = f"{what}: {strerror(status)} (status {status})"
    if status == ELSA_ERR_SHAPE:
        raise ShapeError(msg)
    if status == ELSA_ERR_NUMERICAL:
        raise NumericalError(msg)
    if status == ELSA_ERR_WORKSPACE:
        raise WorkspaceError(msg)
    raise ElsaCudaError(f"{msg}: {lib().elsa_last_cuda_error().decode()}")
