"""INTEGRATION.md's maintainer binding, executed verbatim: the numpy +
ctypes `scan_forward_gpu` block is extracted from the document, its
`scanattn` imports are satisfied by this repository's mirrors of the
reference types (scanattn_compat), and its output is checked against the
FP64 oracle within the reference's bound (verify.py:320-358)."""

import os
import re
import types

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2604_23798_b200 import _lib, scanattn_compat as sc  # noqa: E402
from paper_2604_23798_b200.errors import NumericalError, ShapeError  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _binding():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# scanattn/gpu.py.*?)```", text, re.S).group(1)
    code = re.sub(r"^from \.\S+ import .*$", "", code, flags=re.M)  # supplied below
    mod = types.ModuleType("scanattn_gpu")
    mod.__dict__.update(LIBELSA_PATH=_lib.LIB_PATH, ScanTrace=sc.ScanTrace,
                        scan_depth=sc.scan_depth, NumericalError=NumericalError,
                        ShapeError=ShapeError, Precision=sc.Precision,
                        AttentionOutput=sc.AttentionOutput, Tensor4=sc.Tensor4)
    exec(compile(code, "INTEGRATION.md", "exec"), mod.__dict__)
    return mod


def test_integration_binding_matches_oracle():
    gpu = _binding()
    for (seed, b, h, n, d, dv) in ((11, 1, 1, 1024, 16, 8), (3, 2, 3, 300, 64, 64)):
        Q, K, V = oracle.generate(seed, "regular", b=b, h=h, n=n, d=d, d_v=dv, dtype=np.float32)
        prob = sc.AttentionProblem(sc.Tensor4(Q), sc.Tensor4(K), sc.Tensor4(V))
        out, trace = gpu.scan_forward_gpu(prob, sc.ScanConfig(trace=True))
        err = oracle.row_rel_err(out.Y.data, oracle.naive_attention(Q, K, V))
        assert err.max() <= oracle.bound_threshold(n)
        assert trace.critical_depth == oracle.scan_depth(n, 128)
    with pytest.raises(ShapeError):
        gpu.scan_forward_gpu(prob, sc.ScanConfig(precision=sc.Precision.FP64))


def test_integration_binding_raises_numerical_error():
    gpu = _binding()
    Q, K, V = oracle.generate(5, "regular", b=1, h=1, n=64, d=8, d_v=8, dtype=np.float32)
    prob = sc.AttentionProblem(sc.Tensor4(Q), sc.Tensor4(K), sc.Tensor4(V))
    prob.K.data[0, 0, 1, 0] = np.inf  # bypass the Tensor4 finiteness check
    with pytest.raises(NumericalError):
        gpu.scan_forward_gpu(prob, sc.ScanConfig())
