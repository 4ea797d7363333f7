"""Host-side behaviour of the drop-in that needs no GPU: loud rejection of
everything outside the FP32 CUDA path (no CPU fallback exists)."""

import numpy as np
import pytest
import torch

import paper_2604_23798_b200 as elsa
from paper_2604_23798_b200 import scanattn_compat


def t(*shape, dtype=torch.float32):
    return torch.zeros(*shape, dtype=dtype)


def test_cpu_tensors_are_rejected_not_computed():
    with pytest.raises(elsa.ShapeError, match="no CPU fallback"):
        elsa.scaled_dot_product_attention(t(1, 1, 4, 8), t(1, 1, 4, 8), t(1, 1, 4, 8))


@pytest.mark.parametrize("kw", [dict(attn_mask=t(4, 4)), dict(dropout_p=0.1), dict(is_causal=True)])
def test_non_goals_raise(kw):
    with pytest.raises(elsa.ShapeError):
        elsa.scaled_dot_product_attention(t(1, 1, 4, 8), t(1, 1, 4, 8), t(1, 1, 4, 8), **kw)


def test_unsupported_dtypes_rejected():
    with pytest.raises(elsa.ShapeError, match="float32"):
        elsa.scaled_dot_product_attention(*(t(1, 1, 4, 8, dtype=torch.float64),) * 3)
    with pytest.raises(elsa.ShapeError, match="no CPU fallback"):
        elsa.scaled_dot_product_attention(*(t(1, 1, 4, 64, dtype=torch.bfloat16),) * 3)
    with pytest.raises(elsa.ShapeError, match="share one dtype"):
        elsa.scaled_dot_product_attention(t(1, 1, 4, 64), t(1, 1, 4, 64), t(1, 1, 4, 64, dtype=torch.bfloat16))


def test_errors_mirror_reference_taxonomy():
    assert issubclass(elsa.ShapeError, ValueError)
    assert issubclass(elsa.NumericalError, ArithmeticError)
    assert issubclass(elsa.ElsaLibraryError, ImportError)


def test_shim_rejects_fp64_before_any_device_work():
    T4, P = scanattn_compat.Tensor4, scanattn_compat.Precision
    x = np.zeros((1, 1, 4, 8), np.float32)
    prob = scanattn_compat.AttentionProblem(T4(x), T4(x), T4(x))
    with pytest.raises(elsa.ShapeError):
        scanattn_compat.scan_forward(prob, scanattn_compat.ScanConfig(precision=P.FP64))
    with pytest.raises(elsa.ShapeError):
        scanattn_compat.ScanConfig(block_size=0)
    assert scanattn_compat.scan_depth(16384, 128) == 24
    assert scanattn_compat.depth_cap(16384) == 31


def test_shim_accepts_reference_config_objects_duck_typed():
    # a reference-style config whose precision enum has .value == "fp64"
    class FakePrec:
        value = "fp64"

    class FakeCfg:
        block_size, tile_q, workers, precision, trace = 128, 64, 1, FakePrec(), False

    x = np.zeros((1, 1, 4, 8), np.float32)
    T4 = scanattn_compat.Tensor4
    prob = scanattn_compat.AttentionProblem(T4(x), T4(x), T4(x))
    with pytest.raises(elsa.ShapeError):
        scanattn_compat.scan_forward(prob, FakeCfg())


def test_gqa_fold_validates_heads_and_rejects_cpu():
    # H_q not a multiple of H_kv
    with pytest.raises(elsa.ShapeError, match="multiple"):
        elsa.scaled_dot_product_attention(t(1, 6, 4, 8), t(1, 4, 4, 8), t(1, 4, 4, 8),
                                          enable_gqa=True)
    # key / value head counts differ
    with pytest.raises(elsa.ShapeError, match="same number of heads"):
        elsa.scaled_dot_product_attention(t(1, 4, 4, 8), t(1, 2, 4, 8), t(1, 1, 4, 8),
                                          enable_gqa=True)
    # a valid fold still has no CPU path
    with pytest.raises(elsa.ShapeError, match="no CPU fallback"):
        elsa.scaled_dot_product_attention(t(1, 4, 4, 8), t(1, 2, 4, 8), t(1, 2, 4, 8),
                                          enable_gqa=True)
