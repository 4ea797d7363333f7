"""C-ABI library checks that need no GPU: the in-tree libelsa.so loads,
exports every symbol include/elsa.h declares, and its host-side logic
(depth bound, split planner, argument validation) behaves."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_2604_23798_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "elsa.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(elsa_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    h = _lib.lib()
    declared = header_functions()
    assert declared == sorted(_lib.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(h, name), name
    assert h.elsa_abi_version() == 1


def test_library_is_sm100a():
    # the fatbin must carry sm_100a SASS (no PTX-only / other-arch build)
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_strerror_codes():
    assert _lib.strerror(0) == "ok"
    assert "shape" in _lib.strerror(2)
    assert "normalizer" in _lib.strerror(3)
    assert "unknown" in _lib.strerror(99)


def test_scan_depth_matches_oracle():
    h = _lib.lib()
    for n in (1, 2, 63, 64, 100, 128, 129, 256, 1024, 16384, 65536, 1 << 20):
        for B in (1, 7, 32, 128, 256):
            assert h.elsa_scan_depth(n, B) == oracle.scan_depth(n, B), (n, B)
    assert h.elsa_scan_depth(0, 128) == -1
    assert h.elsa_scan_depth(16, 0) == -1


def _shape(B, H, n_q, n_kv, d=64, dv=64):
    s = _lib.ElsaShape()
    s.B, s.H, s.n_q, s.n_kv, s.d, s.dv = B, H, n_q, n_kv, d, dv
    for arr, w in ((s.q_stride, d), (s.k_stride, d), (s.v_stride, dv), (s.y_stride, dv)):
        arr[0], arr[1], arr[2] = H * max(n_q, n_kv) * w, max(n_q, n_kv) * w, w
    return s


def resolve(s, req=0):
    return _lib.lib().elsa_resolve_kv_splits(ctypes.byref(s), req)


def test_split_planner():
    # big grids need no split; tiny grids split the key range to fill 148 SMs
    assert resolve(_shape(1, 16, 16384, 16384)) == 1
    assert resolve(_shape(8, 12, 512, 512)) <= 2
    s = resolve(_shape(1, 1, 1024, 1024))
    assert 2 <= s <= 16
    # explicit requests are honoured up to the tile count / 32
    assert resolve(_shape(1, 1, 1024, 1024), 4) == 4
    assert resolve(_shape(1, 1, 1024, 1024), 64) == 16
    assert resolve(_shape(1, 1, 100, 10), 8) == 1
    # no empty splits: ceil(tiles / ceil(tiles / s))
    assert resolve(_shape(1, 1, 64, 64 * 10), 4) == 4
    assert resolve(_shape(1, 1, 64, 64 * 10), 7) == 5
    ws = _lib.lib().elsa_workspace_bytes(ctypes.byref(_shape(1, 1, 1024, 1024)), 4)
    assert ws == 4 * 1024 * 66 * 4 + 16  # m | S | 16-byte pad | W


@pytest.mark.parametrize("bad", [
    dict(d=257), dict(dv=4097), dict(dv=0), dict(d=0), dict(n_kv=0),
])
def test_invalid_shapes_rejected_without_touching_the_gpu(bad):
    kw = dict(B=1, H=1, n_q=8, n_kv=8, d=64, dv=64)
    kw.update(bad)
    s = _shape(**kw)
    h = _lib.lib()
    fake = ctypes.c_void_p(16)
    st = h.elsa_fwd_f32(fake, fake, fake, fake, ctypes.byref(s), ctypes.c_double(0.125), 0,
                        None, 0, None)
    assert st == _lib.ELSA_ERR_SHAPE


def test_bad_scale_and_ranges_rejected():
    s = _shape(1, 1, 8, 8)
    h = _lib.lib()
    fake = ctypes.c_void_p(16)
    assert h.elsa_fwd_f32(fake, fake, fake, fake, ctypes.byref(s), ctypes.c_double(np.inf), 0,
                          None, 0, None) == _lib.ELSA_ERR_SHAPE
    assert h.elsa_fwd_f32(fake, fake, fake, fake, ctypes.byref(s), ctypes.c_double(0.1), -1,
                          None, 0, None) == _lib.ELSA_ERR_SHAPE
    assert h.elsa_partial_f32(fake, fake, fake, ctypes.byref(s), ctypes.c_double(0.1), 4, 2,
                              fake, fake, fake, 1, None, 0, None) == _lib.ELSA_ERR_SHAPE
    assert h.elsa_partial_f32(fake, fake, fake, ctypes.byref(s), ctypes.c_double(0.1), 0, 9,
                              fake, fake, fake, 1, None, 0, None) == _lib.ELSA_ERR_SHAPE
    assert h.elsa_merge_f32(fake, fake, fake, 0, 4, 8, 4, 1, fake, None, None, None,
                            None) == _lib.ELSA_ERR_SHAPE
    assert h.elsa_merge_f32(fake, fake, fake, 33, 4, 8, 4, 1, fake, None, None, None,
                            None) == _lib.ELSA_ERR_SHAPE
    assert h.elsa_merge_f32(fake, fake, fake, 2, 4, 4097, 4, 1, fake, None, None, None,
                            None) == _lib.ELSA_ERR_SHAPE
    assert h.elsa_merge_f32(fake, fake, fake, 2, 4, 0, 4, 1, fake, None, None, None,
                            None) == _lib.ELSA_ERR_SHAPE


def test_wide_head_workspace_counts_every_column_slice():
    # dv > 64 runs as ceil(dv / 64) slices; the split workspace keeps
    # 2 + 64 * slices floats per row per split
    h = _lib.lib()
    for d, dv, per_row in ((128, 64, 66), (64, 128, 130), (128, 200, 2 + 256), (96, 1, 66)):
        ws = h.elsa_workspace_bytes(ctypes.byref(_shape(1, 1, 1024, 1024, d=d, dv=dv)), 4)
        assert ws == 4 * 1024 * per_row * 4 + 16, (d, dv, ws)
    assert h.elsa_block_scan_workspace_bytes(10, 5, 200) == 10 * 8 * 202 * 4
    assert h.elsa_block_scan_workspace_bytes(10, 5, 4097) == 0


def test_empty_problem_is_a_noop():
    s = _shape(0, 4, 8, 8)
    h = _lib.lib()
    fake = ctypes.c_void_p(16)
    assert h.elsa_fwd_f32(fake, fake, fake, fake, ctypes.byref(s), ctypes.c_double(0.1), 0,
                          None, 0, None) == 0


def test_host_entry_validates_before_touching_the_device():
    # elsa_fwd_f32_host takes dense host arrays; a non-dense stride or a
    # missing pointer is a ShapeError before any CUDA call
    h = _lib.lib()
    s = _shape(2, 3, 128, 128)
    buf = (ctypes.c_float * 4)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    s.q_stride[2] = 68  # padded rows: not the dense layout
    assert h.elsa_fwd_f32_host(p, p, p, p, ctypes.byref(s), 0.125, 0, None, 0, None) == 2
    s = _shape(2, 3, 128, 128)
    assert h.elsa_fwd_f32_host(None, p, p, p, ctypes.byref(s), 0.125, 0, None, 0, None) == 2
    assert h.elsa_fwd_f32_host(p, p, p, p, ctypes.byref(s), float("nan"), 0, None, 0, None) == 2


def test_peer_merge_validates_before_touching_the_device():
    h = _lib.lib()
    buf = (ctypes.c_float * 4)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    arr = (ctypes.c_void_p * 1)(p)
    y = p
    # 33 chunks > the 32-leaf tree; 0 ranks; rows past rows_total; missing pointers
    assert h.elsa_merge_peers_f32(arr, arr, arr, 1, 33, 4, 0, 4, 64, y, None) == 2
    assert h.elsa_merge_peers_f32(arr, arr, arr, 0, 1, 4, 0, 4, 64, y, None) == 2
    assert h.elsa_merge_peers_f32(arr, arr, arr, 1, 8, 4, 2, 4, 64, y, None) == 2
    assert h.elsa_merge_peers_f32(None, arr, arr, 1, 8, 4, 0, 4, 64, y, None) == 2


def test_describe_plan_names_every_width_configuration():
    h = _lib.lib()
    buf = ctypes.create_string_buffer(128)
    want = {(64, 64): ("w8r8", "w4r8", "w8r16"), (128, 64): ("w8r8d128",), (64, 128): ("w8r8v128",),
            (128, 128): ("w8r8d128v128",), (96, 96): ("w8r8d96v96",), (80, 40): ("w8r8d96",),
            (90, 100): ("w8r8d96v128",), (64, 96): ("w8r8v96",), (128, 80): ("w8r8d128v96",),
            (256, 256): ("w4r8d256v256",),
            (256, 64): ("w8r8d256",), (200, 100): ("w4r8d256v128",), (32, 32): ("w8r8d32v32",),
            (32, 40): ("w8r8", "w4r8", "w8r16")}
    for (d, dv), names in want.items():
        assert h.elsa_describe_plan(ctypes.byref(_shape(1, 16, 4096, 4096, d=d, dv=dv)), 0, buf,
                                    128) == 0
        desc = buf.value.decode()
        assert desc.split()[0] in names, (d, dv, desc)
    assert h.elsa_describe_plan(ctypes.byref(_shape(1, 1, 512, 512, d=128, dv=300)), 0, buf, 128) == 0
    assert "dv_slices=3" in buf.value.decode()
