"""Exception taxonomy of the drop-in, mirroring the reference's
``scanattn.errors`` (/root/reference/pkg/src/scanattn/errors.py:8-29) so the
same ``except`` clauses work; the C-ABI status codes map onto these
(include/elsa.h: 2 -> ShapeError, 3 -> NumericalError)."""


class ShapeError(ValueError):
    """Inconsistent dimensions or invalid configuration (errors.py:8)."""


class NumericalError(ArithmeticError):
    """Zero / non-finite softmax normalizer or NaN state (errors.py:12)."""


class WorkspaceError(RuntimeError):
    """The caller-provided workspace is missing or too small."""


class ElsaCudaError(RuntimeError):
    """A CUDA runtime / launch failure inside libelsa."""


class ElsaLibraryError(ImportError):
    """libelsa.so is missing or unloadable; there is no CPU fallback."""


class TensorFileError(Exception):
    """ATN1 tensor-file format violation (errors.py:32)."""


class BadMagicError(TensorFileError):
    """Not an ATN1 file (errors.py:36)."""


class BadVersionError(TensorFileError):
    """Unsupported ATN1 version (errors.py:40)."""


class BadDtypeError(TensorFileError):
    """Unknown ATN1 dtype code (errors.py:44)."""


class TruncatedPayloadError(TensorFileError):
    """Payload shorter than the header promises, or bad trailer (errors.py:48)."""


class DimsMismatchError(TensorFileError):
    """Payload length disagrees with the dims (errors.py:53)."""
