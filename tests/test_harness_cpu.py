"""Host-side harness mirrors, pinned to the
reference's own outputs (tests/golden/harness.npz, made by
tests/golden/make_golden_blocks.py): ATN1 files byte-for-byte, the
scanattn-bench-v1 report JSON/CSV byte-for-byte, the scaling fit and the
nearest-rank percentiles."""

import json
import os

import numpy as np
import pytest

from paper_2604_23798_b200 import errors, report, tensorio


@pytest.mark.parametrize("tag", ["f32", "f64"])
def test_atn1_bytes_match_reference(golden, tmp_path, tag):
    z = golden["harness"]
    path = tmp_path / "t.atn"
    tensorio.write_tensor(str(path), z[f"atn1_{tag}_data"])
    assert path.read_bytes() == z[f"atn1_{tag}_bytes"].tobytes()
    back = tensorio.read_tensor(str(path))
    assert back.dtype == z[f"atn1_{tag}_data"].dtype
    assert np.array_equal(back, z[f"atn1_{tag}_data"])


def test_atn1_torch_input(tmp_path):
    torch = pytest.importorskip("torch")
    t = torch.randn(1, 2, 3, 4)
    p = tmp_path / "y.atn"
    tensorio.write_tensor(str(p), t)
    assert np.array_equal(tensorio.read_tensor(str(p)), t.numpy())


def test_atn1_errors(golden, tmp_path):
    good = golden["harness"]["atn1_f32_bytes"].tobytes()
    p = tmp_path / "bad.atn"
    cases = [
        (b"XXXX" + good[4:], errors.BadMagicError),
        (good[:8] + (2).to_bytes(4, "little") + good[12:], errors.BadVersionError),
        (good[:12] + bytes([7]) + good[13:], errors.BadDtypeError),
        (good[:-12], errors.TruncatedPayloadError),
        (good[:-8] + b"\0\0\0\0" + good[-8:], errors.DimsMismatchError),
        (good[:-8] + (1).to_bytes(8, "little"), errors.TruncatedPayloadError),
    ]
    for raw, exc in cases:
        p.write_bytes(raw)
        with pytest.raises(exc):
            tensorio.read_tensor(str(p))
    with pytest.raises(errors.ShapeError):
        tensorio.write_tensor(str(p), np.zeros((2, 2), np.float32))
    with pytest.raises(errors.ShapeError):
        tensorio.write_tensor(str(p), np.zeros((1, 1, 2, 2), np.float16))


def test_report_bytes_match_reference(golden, tmp_path):
    """The writer is byte-equal to the reference's report (records, fit
    serialisation, CSV) when given the reference's fit coefficients; the fit
    itself (an independent QR solve) agrees to ~1e-14 relative."""
    z = golden["harness"]
    rec = report.BenchRecord(mode="scan", n=1024, block_size=128, tile_q=64, d=64, d_v=64,
                             b=1, h=16, precision="fp32", repeats=5, warmup=2,
                             latencies=[3.0e-4, 2.5e-4, 2.7e-4, 2.6e-4, 2.9e-4],
                             merge_count=123, leaf_count=456, peak_extra_memory=789)
    pts = [tuple(p) for p in z["fit_pts"]]
    a, b, c, res = (float(x) for x in z["fit_coef"])
    fit = report.ScalingFit(a, b, c, res, 128, pts)
    jp, cp = report.emit_report([rec], [fit], str(tmp_path / "r.json"))
    with open(jp, "rb") as f:
        assert f.read() == z["report_json"].tobytes()
    with open(cp, "rb") as f:
        assert f.read() == z["report_csv"].tobytes()
    assert cp == str(tmp_path / "r.csv")
    # our own fit, serialised: same document up to the fit's last bits
    jp2, _ = report.emit_report([rec], [report.fit_scaling(pts, 128)], str(tmp_path / "s.json"))
    with open(jp2) as f:
        ours = json.load(f)
    ref = json.loads(z["report_json"].tobytes())
    assert ours["records"] == ref["records"] and ours["schema"] == ref["schema"]
    for key in ("a", "b", "c", "residual"):
        assert ours["fits"][0][key] == pytest.approx(ref["fits"][0][key], rel=1e-11)
    assert ours["fits"][0]["points"] == ref["fits"][0]["points"]


def test_fit_and_percentiles(golden):
    z = golden["harness"]
    fit = report.fit_scaling([tuple(p) for p in z["fit_pts"]], 128)
    np.testing.assert_allclose([fit.a, fit.b, fit.c, fit.residual], z["fit_coef"], rtol=1e-11)
    pc = report.nearest_rank_percentiles(z["pct_in"])
    assert np.array_equal(np.array([pc["median"], pc["p95"], pc["p99"]]), z["pct_out"])
    # exact synthetic data is recovered
    pts = [(n, 0.01 * report._depth(n, 128) + 2e-9 * n * n + 0.5) for n in (1024, 2048, 4096, 8192)]
    f = report.fit_scaling(pts, 128)
    assert abs(f.a - 0.01) < 1e-9 and abs(f.b - 2e-9) < 1e-15 and abs(f.c - 0.5) < 1e-8
    assert f.residual < 1e-12
    assert abs(f.predict(16384) - (0.01 * 24 + 2e-9 * 16384 ** 2 + 0.5)) < 1e-6
    with pytest.raises(errors.ShapeError):
        report.fit_scaling([(1024, 1.0), (1024, 2.0), (2048, 3.0)], 128)
    with pytest.raises(errors.ShapeError):
        report.run_bench(1, 1, 64, mode="naive")
