"""Pin the numpy oracle to the real reference via the committed golden fixtures.

The fixtures were produced by running /root/reference's own `eikfld` package
(tests/golden/make_golden.py).  The oracle restates the same arithmetic, so
agreement is asserted bit for bit (np.array_equal) wherever the reference
returns the value directly.
"""

import math

import numpy as np
import pytest

import eikfld_oracle as orc
from conftest import load_golden


def test_engine_kats_bit_exact():
    g = load_golden("engine_12x10.npz")
    counts = tuple(g["counts"])
    k = orc.kernel_exp(counts, float(g["spacing"]), float(g["tau"]))
    assert np.array_equal(k, g["kernel"])
    cv = orc.Convolver(counts, k.shape)
    assert np.array_equal(cv.convolve(k, g["dense"].reshape(counts)).reshape(-1), g["conv_dense"])
    many = cv.convolve_many([k, g["k2"], k * 0.25], g["impulses"].reshape(counts))
    for i in range(3):
        assert np.array_equal(many[i].reshape(-1), g[f"many{i}"])


def test_line_bit_exact():
    g = load_golden("line_9.npz")
    counts = tuple(g["counts"])
    s = orc.s_fft(g["nodes"], counts, float(g["spacing"]), float(g["tau"]))
    assert np.array_equal(s, g["S"])
    # tests/test_distance.py:91-97 known answer
    assert abs(s[4] - (0.2 - 0.05 * math.log(2.0))) < 1e-13
    den, (sx,) = orc.gradient_unchecked(g["nodes"], counts, float(g["spacing"]), float(g["tau"]))
    assert np.array_equal(sx, g["Sx"])


def test_field64_bit_exact():
    g = load_golden("field_64.npz")
    counts, h, tau = tuple(g["counts"]), float(g["spacing"]), float(g["tau"])
    assert np.array_equal(orc.s_fft(g["nodes"], counts, h, tau), g["S"])
    _, (sx, sy) = orc.gradient_unchecked(g["nodes"], counts, h, tau)
    assert np.array_equal(sx, g["Sx"]) and np.array_equal(sy, g["Sy"])
    _, sxx, syy, sxy = orc.hessian_2d_unchecked(g["nodes"], counts, h, tau)
    for a, b in ((sxx, "Sxx"), (syy, "Syy"), (sxy, "Sxy")):
        assert np.array_equal(a, g[b])
    pts = orc.coords_of_flat(g["nodes"], (0.0, 0.0), h, counts)
    assert np.array_equal(orc.s_direct(pts, (0.0, 0.0), h, counts, tau), g["S_direct"])


def test_winding_bit_exact():
    g = load_golden("winding_128.npz")
    counts, h, origin = tuple(g["counts"]), float(g["spacing"]), tuple(g["origin"])
    mu, flagged = orc.winding_field(g["vertices"], origin, h, counts)
    assert np.array_equal(mu, g["mu"])
    assert np.array_equal(flagged, g["flagged"])
    mask = orc.classify(mu, flagged, counts, "winding2d")
    assert np.array_equal(mask, g["mask"])
    assert 0.2 < mask.mean() < 0.5


def test_volume_bit_exact():
    g = load_golden("vol_24.npz")
    counts, h, origin, tau = tuple(g["counts"]), float(g["spacing"]), tuple(g["origin"]), float(g["tau"])
    assert np.array_equal(orc.s_fft(g["nodes"], counts, h, tau), g["S"])
    _, grads = orc.gradient_unchecked(g["nodes"], counts, h, tau)
    for a, name in zip(grads, ("Sx", "Sy", "Sz")):
        assert np.array_equal(a, g[name])
    mu, flagged = orc.degree_field(g["triangles"], g["centers"], g["normals"], origin, h, counts)
    assert np.array_equal(mu, g["mu"])
    assert np.array_equal(orc.classify(mu, flagged, counts, "degree3d"), g["mask"])


@pytest.mark.slow
def test_c1_bit_exact():
    g = load_golden("c1.npz")
    counts, tau = tuple(g["counts"]), float(g["tau"])
    assert np.array_equal(orc.s_fft(g["nodes"], counts, 1.0, tau), g["S"])
    _, (sx, sy) = orc.gradient_unchecked(g["nodes"], counts, 1.0, tau)
    assert np.array_equal(sx, g["Sx"]) and np.array_equal(sy, g["Sy"])
    # reference vs exact soft-min on C1 is ~1.9e-6
    err = np.abs(g["S"] - g["S_direct"]).max()
    assert 1e-7 < err < 1e-5


def test_c5_item_subsample_bit_exact():
    g = load_golden("c5_item0_sub.npz")
    counts = (512, 512)
    out = orc.run_config_unchecked(g["nodes"], counts, 1.0, 0.5)
    sel = g["sel"]
    assert np.array_equal(out["phi"][sel], g["phi"])
    assert np.array_equal(out["grad"][0][sel], g["Sx"])
    assert np.array_equal(out["grad"][1][sel], g["Sy"])
    assert int((out["phi"] <= 0).sum()) == int(g["phi_le0"]) > 0  # the reference raises (T4)


def test_oracle_raises_on_underflow():
    # tests/test_distance.py:117-122
    with pytest.raises(orc.OracleUnderflow, match="precision"):
        orc.s_fft([0], (32, 32), 0.1, 1e-4)


def test_bigfloat_fixtures_match_direct_mp_sum():
    """The reference's big-float FFT answers (p = 200, tests/golden/
    make_golden_bigfloat.py) equal the exact direct sums of the sampled
    kernel: the truth the double-double GPU path is checked against."""
    for name in ("bigfloat_1d", "bigfloat_2d", "bigfloat_3d"):
        g = load_golden(f"{name}.npz")
        ref = orc.phi_direct_mp(g["nodes"], g["counts"], float(g["h"]), float(g["tau"]), dps=50)
        assert np.abs(ref - g["log10_phi"]).max() <= 1e-12, name
        assert g["log10_phi"].min() < -22  # far below the float64 round-off floor
