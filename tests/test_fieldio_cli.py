"""EIKFLD01 writer/reader byte-compatible with the reference, and the CLI front end."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO

from paper_1112_3010_b200 import GridSpec, PrecisionConfig, ScalarField, ValidationError, fieldio


def _sample():
    g = GridSpec(origin=(-0.5, 0.25, 1.0), spacing=0.125, counts=(4, 5, 6))
    vals = np.random.Generator(np.random.PCG64(8)).standard_normal(g.num_nodes)
    return ScalarField(g, vals, flagged_nodes=[3, 77])


def test_bytes_identical_to_reference_writer(tmp_path):
    p = str(tmp_path / "s.fld")
    fieldio.write_field(p, _sample(), "S", PrecisionConfig.native64(0.1), {"method": "fft", "k": 1})
    assert open(p, "rb").read() == open(os.path.join(GOLDEN, "ref_field.fld"), "rb").read()


def test_roundtrip_and_header(tmp_path):
    p = str(tmp_path / "s.fld")
    f = _sample()
    fieldio.write_field(p, f, "S", PrecisionConfig.bigfloat(2.5e-4, 512), {"method": "fft"})
    header, back = fieldio.read_field(p)
    assert np.array_equal(back.values, f.values) and back.grid == f.grid
    assert header["precision"] == "big:512" and header["precision_bits"] == 512
    assert list(back.flagged_nodes) == [3, 77]
    header2, ref = fieldio.read_field(os.path.join(GOLDEN, "ref_field.fld"))
    assert np.array_equal(ref.values, f.values) and header2["params"] == {"k": 1, "method": "fft"}


def test_rejects_bad_magic(tmp_path):
    p = tmp_path / "bad.fld"
    p.write_bytes(b"NOTAFILE" + b"\x00" * 32)
    with pytest.raises(ValidationError):
        fieldio.read_header(str(p))


def _cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_1112_3010_b200.cli", *args], cwd=cwd or REPO,
                          capture_output=True, text=True, env={**os.environ, "PYTHONPATH": REPO})


def test_cli_errors_exit_2(tmp_path):
    r = _cli("dt", "--min", "0,0", "--counts", "8,8", "--spacing", "1", "--tau", "1", "--out", str(tmp_path / "a"))
    assert r.returncode == 2 and r.stderr.startswith("error:")
    pts = tmp_path / "p.csv"
    pts.write_text("1,1\n")
    r = _cli("dt", "--points", str(pts), "--min", "0,0", "--counts", "8,8", "--spacing", "1", "--tau", "1",
             "--method", "exact", "--out", str(tmp_path / "a"))
    assert r.returncode == 2 and "reference" in r.stderr
    r = _cli("info", str(tmp_path / "missing.fld"))
    assert r.returncode == 2


@pytest.mark.gpu
def test_cli_dt_grad_sign_on_gpu(cuda_ok, tmp_path):
    import eikfld_oracle as orc

    pts = np.array([[3.0, 4.0], [10.0, 2.0], [7.0, 12.0]])
    (tmp_path / "p.csv").write_text("\n".join(f"{x},{y}" for x, y in pts))
    common = ["--points", str(tmp_path / "p.csv"), "--min", "0,0", "--counts", "16,16", "--spacing", "1",
              "--tau", "1.5"]
    assert _cli("dt", *common, "--out", str(tmp_path / "S.fld")).returncode == 0
    assert _cli("grad", *common, "--out-prefix", str(tmp_path / "g_")).returncode == 0
    nodes = orc.snap(pts, (0.0, 0.0), 1.0, (16, 16))
    ref = orc.run_config_unchecked(np.unique(nodes), (16, 16), 1.0, 1.5)
    hdr, S = fieldio.read_field(str(tmp_path / "S.fld"))
    assert hdr["field"] == "S" and hdr["tau"] == 1.5
    assert np.abs(S.values - ref["S"]).max() <= 1e-9 * np.abs(ref["S"]).max()
    _, gx = fieldio.read_field(str(tmp_path / "g_S_x.fld"))
    keep = np.ones(256, bool)
    keep[np.unique(nodes)] = False
    assert np.abs(gx.values - ref["grad"][0])[keep].max() <= 1e-9
    th = np.linspace(0, 2 * np.pi, 60, endpoint=False)
    (tmp_path / "c.csv").write_text("\n".join(f"{7.5 + 5 * np.cos(t)},{7.5 + 5 * np.sin(t)}" for t in th))
    r = _cli("sign", "--curve", str(tmp_path / "c.csv"), "--min", "0,0", "--counts", "16,16", "--spacing", "1",
             "--mu-out", str(tmp_path / "mu.fld"), "--mask-out", str(tmp_path / "mask.fld"),
             "--distance-field", str(tmp_path / "S.fld"), "--signed-out", str(tmp_path / "sS.fld"))
    assert r.returncode == 0, r.stderr
    _, mu = fieldio.read_field(str(tmp_path / "mu.fld"))
    mu_ref, fl = orc.winding_field(np.stack([7.5 + 5 * np.cos(th), 7.5 + 5 * np.sin(th)], 1), (0.0, 0.0), 1.0,
                                   (16, 16))
    assert np.abs(mu.values - mu_ref).max() <= 1e-12
    _, mask = fieldio.read_field(str(tmp_path / "mask.fld"))
    assert np.array_equal(mask.values, orc.classify(mu_ref, fl, (16, 16), "winding2d"))
    info = _cli("info", str(tmp_path / "mask.fld"))
    assert info.returncode == 0 and json.loads(info.stdout)["field"] == "mask"
