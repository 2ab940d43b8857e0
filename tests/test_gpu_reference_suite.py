"""The reference's own fp64 unit tests, run against this build.

R/pkg/tests/test_convolution.py, test_distance.py, test_derivatives.py and
test_sign.py (staged by tools/stage_reftests.py into oracle/_ref/reftests/)
run with `import eikfld` aliased to paper_1112_3010_b200 (tests/
reftest_support.py).  Every test except the big-float ones listed in
reftest_support.DESELECT must pass.  The GPU test runs them on the device;
the CPU test checks that the aliased suite imports and collects.
"""

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

import reftest_support as rs

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(args, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([HERE, os.path.join(rs.REPO, "oracle"), rs.REPO, env.get("PYTHONPATH", "")])
    xml = os.path.join(str(tmp_path), "ref.xml")
    cmd = [sys.executable, "-m", "pytest", "-p", "reftest_support", "-p", "no:cacheprovider", "-q",
           f"--junitxml={xml}", *args, *[os.path.join(rs.STAGE, f) for f in rs.FILES]]
    p = subprocess.run(cmd, cwd=rs.REPO, env=env, capture_output=True, text=True, timeout=1800)
    return p, xml


def _staged():
    if not all(os.path.exists(os.path.join(rs.STAGE, f)) for f in rs.FILES + ("shapes.py",)):
        pytest.skip("reference tests not staged (tools/stage_reftests.py needs /root/reference)")


def test_reference_suite_collects(tmp_path):
    _staged()
    p, _ = _run(["--collect-only"], tmp_path)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert f"({len(rs.DESELECT)} deselected)" in p.stdout, p.stdout[-2000:]


@pytest.mark.gpu
def test_reference_fp64_suite_passes(cuda_ok, tmp_path):
    _staged()
    p, xml = _run([], tmp_path)
    root = ET.parse(xml).getroot()
    cases = root.iter("testcase")
    failed, passed = [], []
    for c in cases:
        name = f"{c.get('classname')}::{c.get('name')}"
        bad = [x for x in c if x.tag in ("failure", "error")]
        skipped = [x for x in c if x.tag == "skipped"]
        if bad:
            failed.append((name, bad[0].get("message", "")[:300]))
        elif not skipped:
            passed.append(name)
    print(f"reference suite: {len(passed)} passed, {len(failed)} failed, {len(rs.DESELECT)} deselected (big-float)")
    assert not failed, failed
    assert len(passed) >= 70, (len(passed), p.stdout[-2000:])
