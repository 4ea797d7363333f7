"""ATN1 tensor files for GPU outputs.

The reference's harness exchanges tensors as ATN1 files
(/root/reference/pkg/src/scanattn/tensorio.py:37-41, 198-239):

    header  "<8sIB4I": magic b"ATN1\\r\\n\\x1a\\n", u32 version 1,
            u8 dtype code (0 = little-endian f32, 1 = f64), u32 dims[4]
    payload the (b, h, n, width) array, C order, little-endian
    trailer u64 payload byte count

``write_tensor`` lets a GPU result (a CUDA or CPU torch tensor, a numpy array
or a ``Tensor4``) be handed to ``scanattn verify --candidate FILE``
(cli.py:155-158); ``read_tensor`` reads any ATN1 file back bit-exactly and
raises the reference's error taxonomy on malformed input.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import (
    BadDtypeError,
    BadMagicError,
    BadVersionError,
    DimsMismatchError,
    ShapeError,
    TruncatedPayloadError,
)

__all__ = ["MAGIC", "VERSION", "write_tensor", "read_tensor"]

MAGIC = b"ATN1\r\n\x1a\n"
VERSION = 1
_HEADER = struct.Struct("<8sIB4I")
_TRAILER = struct.Struct("<Q")
_DTYPES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


def _as_numpy(t):
    data = getattr(t, "data", t)
    if hasattr(data, "detach") and hasattr(data, "cpu"):  # torch tensor
        data = data.detach().cpu().numpy()
    arr = np.asarray(data)
    if arr.ndim != 4:
        raise ShapeError(f"ATN1 holds (b, h, n, width) tensors, got shape {arr.shape}")
    if arr.dtype == np.float32:
        code = 0
    elif arr.dtype == np.float64:
        code = 1
    else:
        raise ShapeError(f"ATN1 stores float32 or float64, got {arr.dtype}")
    if any(x >= 1 << 32 for x in arr.shape):
        raise ShapeError("ATN1 dims are u32")
    return code, arr


def write_tensor(path, t):
    """Serialize ``t`` as ATN1 (tensorio.py:198-206)."""
    code, arr = _as_numpy(t)
    payload = np.ascontiguousarray(arr, dtype=_DTYPES[code]).tobytes()
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, VERSION, code, *arr.shape))
        f.write(payload)
        f.write(_TRAILER.pack(len(payload)))


def read_tensor(path):
    """Read an ATN1 file into a native-endian numpy array (tensorio.py:209-239)."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HEADER.size or raw[:8] != MAGIC:
        raise BadMagicError(f"{path}: not an ATN1 file")
    _, version, code, *dims = _HEADER.unpack_from(raw)
    if version != VERSION:
        raise BadVersionError(f"{path}: version {version}, expected {VERSION}")
    if code not in _DTYPES:
        raise BadDtypeError(f"{path}: unknown dtype code {code}")
    dt = _DTYPES[code]
    expected = int(np.prod(dims, dtype=np.int64)) * dt.itemsize
    body = raw[_HEADER.size:]
    if len(body) < expected + _TRAILER.size:
        raise TruncatedPayloadError(
            f"{path}: payload has {max(len(body) - 8, 0)} bytes, header promises {expected}")
    if len(body) != expected + _TRAILER.size:
        raise DimsMismatchError(
            f"{path}: payload length {len(body) - 8} disagrees with dims {tuple(dims)}")
    (trailer,) = _TRAILER.unpack_from(body, expected)
    if trailer != expected:
        raise TruncatedPayloadError(f"{path}: trailing byte count {trailer} != payload length {expected}")
    data = np.frombuffer(body[:expected], dtype=dt).reshape(dims)
    return data.astype(data.dtype.newbyteorder("="), copy=True)
