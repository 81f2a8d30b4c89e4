"""PLY I/O against fixtures written / read by the reference
(oracle/gen_golden_ply.py, sc/asset.py:178-321)."""

import os
import tempfile

import numpy as np
import pytest

from conftest import ROOT

import paper_2511_19202_b200 as sc
from paper_2511_19202_b200.asset import Asset

Z = np.load(os.path.join(ROOT, "tests", "golden", "ply_cases.npz"))
FIELDS = ("means", "log_scales", "rotations", "opacity_logits", "sh_coeffs")


def _asset(prefix, deg):
    return Asset(*(Z[f"{prefix}_{k}"] for k in FIELDS), sh_degree=deg)


@pytest.mark.parametrize("deg", [0, 1, 3])
def test_save_matches_reference_bytes_and_roundtrips(deg, tmp_path):
    a = _asset(f"asset_deg{deg}", deg)
    p = tmp_path / "a.ply"
    sc.save_ply(a, p)
    assert p.read_bytes() == Z[f"saved_deg{deg}"].tobytes()
    b = sc.load_ply(p)
    assert b.sh_degree == deg
    for k in FIELDS:
        np.testing.assert_array_equal(getattr(b, k), getattr(a, k))


def test_load_foreign_file_like_reference(tmp_path):
    p = tmp_path / "f.ply"
    p.write_bytes(Z["foreign_raw"].tobytes())
    a = sc.load_ply(p)
    for k in FIELDS:
        np.testing.assert_array_equal(getattr(a, k), Z[f"foreign_{k}"], err_msg=k)


@pytest.mark.parametrize("mutate, msg", [
    (lambda r: b"plx" + r[3:], "malformed PLY header"),
    (lambda r: r.replace(b"binary_little_endian", b"ascii"), "expected binary_little_endian"),
    (lambda r: r.replace(b"property float opacity\n", b""), "missing property opacity"),
    (lambda r: r.replace(b"property float x\n", b"property list uchar int x\n"), "list properties"),
    (lambda r: r.replace(b"property float x\n", b"property half x\n"), "unsupported property type"),
    (lambda r: r[:-10], "truncated body"),
])
def test_malformed_files_raise(mutate, msg, tmp_path):
    p = tmp_path / "bad.ply"
    p.write_bytes(mutate(Z["saved_deg0"].tobytes()))
    with pytest.raises(ValueError, match=msg):
        sc.load_ply(p)


def test_zero_quaternion_and_non_finite(tmp_path):
    a = _asset("asset_deg0", 0)
    q = a.rotations.copy()
    q[3] = 0.0
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "z.ply")
        sc.save_ply(Asset(a.means, a.log_scales, q, a.opacity_logits, a.sh_coeffs, 0), p)
        with pytest.raises(ValueError, match="zero-norm"):
            sc.load_ply(p)
        m = a.means.copy()
        m[0, 0] = np.nan
        sc.save_ply(Asset(m, a.log_scales, a.rotations, a.opacity_logits, a.sh_coeffs, 0), p)
        with pytest.raises(ValueError, match="non-finite value in position"):
            sc.load_ply(p)
