"""ATN1 tensor files for GPU outputs.

The reference's harness exchanges (b, h, n, width) tensors as ATN1 files; the
format (tensorio.py:37-41, 198-239 of the reference) is

    offset 0   8 bytes  magic b"ATN1\\r\\n\\x1a\\n"
    offset 8   u32      format version (1)
    offset 12  u8       element code: 0 = float32, 1 = float64
    offset 13  4 x u32  dims (b, h, n, width)
    offset 29  payload  C-order elements, little endian
    end - 8    u64      payload length in bytes

all little endian. :func:`write_tensor` lets a GPU result (a CUDA or CPU
torch tensor, a numpy array or anything with a ``.data`` array such as the
reference's ``Tensor4``) be handed to ``scanattn verify --candidate FILE``
(cli.py:155-158); :func:`read_tensor` validates a file section by section
(magic, version, element code, then the payload length against the dims and
the trailer) and raises the reference's error classes, so callers' ``except``
clauses keep working.
"""

from __future__ import annotations

import os
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
_PREAMBLE = struct.Struct("<8sIB4I")      # magic, version, code, dims
_LENGTH = struct.Struct("<Q")             # trailing payload byte count
_ELEMENT = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_CODE = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
_U32_LIMIT = 1 << 32


def _host_array(t):
    """numpy view of a torch tensor (any device), a numpy array or an object
    carrying one in ``.data``."""
    inner = t.data if hasattr(t, "data") and not isinstance(t, np.ndarray) else t
    if hasattr(inner, "detach"):                     # torch.Tensor
        inner = inner.detach().to("cpu").numpy()
    return np.asarray(inner)


def write_tensor(path, t):
    """Serialize a (b, h, n, width) float32/float64 tensor as ATN1."""
    arr = _host_array(t)
    code = _CODE.get(arr.dtype)
    if arr.ndim != 4:
        raise ShapeError(f"an ATN1 file stores a rank-4 (b, h, n, width) tensor; "
                         f"this one has shape {arr.shape}")
    if code is None:
        raise ShapeError(f"ATN1 element types are float32 and float64, not {arr.dtype}")
    if max(arr.shape) >= _U32_LIMIT:
        raise ShapeError(f"dims {arr.shape} exceed the u32 fields of the ATN1 header")
    payload = np.ascontiguousarray(arr).astype(_ELEMENT[code], copy=False).tobytes()
    blob = b"".join((_PREAMBLE.pack(MAGIC, VERSION, code, *arr.shape), payload,
                     _LENGTH.pack(len(payload))))
    with open(path, "wb") as fh:
        fh.write(blob)


def read_tensor(path):
    """Read an ATN1 file into a native-endian numpy array, bit-exactly."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_PREAMBLE.size)
        if len(head) < _PREAMBLE.size or not head.startswith(MAGIC):
            raise BadMagicError(f"{path}: missing the ATN1 signature")
        _, version, code, *dims = _PREAMBLE.unpack(head)
        if version != VERSION:
            raise BadVersionError(f"{path}: ATN1 format version {version} is not supported "
                                  f"(this reader handles {VERSION})")
        elem = _ELEMENT.get(code)
        if elem is None:
            raise BadDtypeError(f"{path}: element code {code} is neither 0 (f32) nor 1 (f64)")
        want = elem.itemsize
        for x in dims:
            want *= x
        have = size - _PREAMBLE.size - _LENGTH.size
        if have < want:
            raise TruncatedPayloadError(f"{path}: dims {tuple(dims)} need {want} payload bytes, "
                                        f"the file holds {max(have, 0)}")
        if have > want:
            raise DimsMismatchError(f"{path}: {have - want} bytes beyond the payload that dims "
                                    f"{tuple(dims)} describe")
        data = np.fromfile(fh, dtype=elem, count=want // elem.itemsize)
        (recorded,) = _LENGTH.unpack(fh.read(_LENGTH.size))
    if recorded != want:
        raise TruncatedPayloadError(f"{path}: trailer records {recorded} payload bytes, "
                                    f"dims give {want}")
    return data.reshape(dims).astype(elem.newbyteorder("="))
