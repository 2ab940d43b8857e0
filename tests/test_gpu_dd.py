"""GPU: the double-double convolution through the
drop-in API with big-float configs, against the REFERENCE's own big-float
pipeline (p = 200, tests/golden/make_golden_bigfloat.py; pinned to exact
direct sums by tests/test_oracle_golden.py).

Tolerance (float64 outputs): |delta| <= 1e-9 * max(|ref|, 1) on every node
with phi / max(phi) >= 1e-20 -- the band the float64 path cannot reach (its
FFT round-off floor is ~1e-16 of max phi), checked below as well."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

BAND = -20.0  # log10(phi / max phi): DD round-off ~1e-30 of max phi -> <= 1e-10 relative here
TOL = 1e-9


def _case(name):
    from paper_1112_3010_b200 import GridSpec, PointSet

    g = load_golden(f"{name}.npz")
    grid = GridSpec(tuple(float(x) for x in g["origin"]), float(g["h"]), tuple(int(c) for c in g["counts"]))
    ps = PointSet.from_node_indices(grid, g["nodes"])
    keep = g["log10_phi"] - g["log10_phi"].max() >= BAND
    return g, grid, ps, keep


def _err(a, b, keep):
    return float((np.abs(a - b)[keep] / np.maximum(np.abs(b[keep]), 1.0)).max())


@pytest.mark.parametrize("name", ["bigfloat_1d", "bigfloat_2d", "bigfloat_3d"])
def test_dd_matches_reference_bigfloat(cuda_ok, name):
    from paper_1112_3010_b200 import PrecisionConfig
    from paper_1112_3010_b200.derivatives import gradient, hessian_2d
    from paper_1112_3010_b200.distance import phi_fft, s_fft

    g, grid, ps, keep = _case(name)
    cfg = PrecisionConfig.bigfloat(float(g["tau"]), 106)
    assert keep.mean() >= 0.75  # most of the grid lies in the checked band ...
    assert (keep & (g["log10_phi"] - g["log10_phi"].max() < -14)).sum() >= 3  # ... incl. nodes float64 cannot resolve
    S = s_fft(ps, grid, cfg).values
    assert _err(S, g["S"], keep) <= TOL
    phi = phi_fft(ps, grid, cfg).values
    assert np.abs(np.log10(phi) - g["log10_phi"])[keep].max() <= 1e-9
    v = gradient(ps, grid, cfg)
    for a, comp in enumerate(v.components):
        assert _err(comp.values, g[f"g{a}"], keep) <= TOL
    if "hxx" in g:
        for got, key in zip(hessian_2d(ps, grid, cfg), ("hxx", "hyy", "hxy")):
            assert _err(got.values, g[key], keep) <= TOL


def test_float64_path_cannot_reach_the_band(cuda_ok):
    """Same inputs through the float64 path: it raises PrecisionError (phi <= 0
    somewhere) or misses the tolerance on the far nodes -- the reason the
    extended-precision path exists (§3.2)."""
    from paper_1112_3010_b200 import PrecisionConfig, PrecisionError, engine
    from paper_1112_3010_b200.distance import s_fft

    g, grid, ps, keep = _case("bigfloat_2d")
    with pytest.raises(PrecisionError):
        s_fft(ps, grid, PrecisionConfig.native64(float(g["tau"])))
    out = engine.DistanceTransform(grid, float(g["tau"]), grad=False).run_host(ps.distinct_nodes())
    ok = keep & np.isfinite(out["S"])
    assert out["n_underflow"] > 0 or _err(out["S"], g["S"], ok) > 1e-6


def test_dd_validation(cuda_ok):
    from paper_1112_3010_b200 import GridSpec, PointSet, PrecisionConfig, ValidationError
    from paper_1112_3010_b200.distance import s_fft

    grid = GridSpec((0.0, 0.0), 1.0, (4096, 8))
    ps = PointSet.from_node_indices(grid, [0])
    with pytest.raises(ValidationError):  # axes up to 2048 nodes
        s_fft(ps, grid, PrecisionConfig.bigfloat(1.0, 106))


# Mirrors of the reference's big-float unit tests at double-double precision
# (R/../tests/test_distance.py:79-89, 179-189; there at p = 192, here p = 106).


def _nodes(grid, seed, k):
    return np.sort(np.random.Generator(np.random.PCG64(seed)).choice(grid.num_nodes, k, replace=False))


def test_k1_recovers_distance_bigfloat(cuda_ok):
    """One source at the centre of a 20 x 20 grid, tau = 0.02: S equals the
    exact Euclidean distance to 1e-12 (R/tests/test_distance.py:87-89)."""
    from paper_1112_3010_b200 import GridSpec, PointSet, PrecisionConfig
    from paper_1112_3010_b200.distance import s_fft

    grid = GridSpec((0.0, 0.0), 0.05, (20, 20))
    ps = PointSet.from_node_indices(grid, [10 * 20 + 10])
    s = s_fft(ps, grid, PrecisionConfig.bigfloat(0.02, 106)).values
    ij = np.stack(np.unravel_index(np.arange(400), (20, 20)), axis=1)
    r = 0.05 * np.sqrt(((ij - np.array([10, 10])) ** 2).sum(axis=1))
    assert np.abs(s - r).max() < 1e-12


@pytest.mark.parametrize("counts", [(40,), (12, 14), (6, 7, 8)])
def test_dimension_independence_bigfloat(cuda_ok, counts):
    """Same pipeline for D = 1, 2, 3 against the stable direct soft-min
    (R/tests/test_distance.py:179-189, tolerance 1e-11)."""
    import eikfld_oracle as orc

    from paper_1112_3010_b200 import GridSpec, PointSet, PrecisionConfig
    from paper_1112_3010_b200.distance import s_fft

    origin = tuple(0.0 for _ in counts)
    grid = GridSpec(origin, 0.02, counts)
    nodes = _nodes(grid, 21, 5)
    ps = PointSet.from_node_indices(grid, nodes)
    s = s_fft(ps, grid, PrecisionConfig.bigfloat(0.05, 106)).values
    pts = np.stack(np.unravel_index(nodes, counts), axis=1) * 0.02
    direct = orc.s_direct(pts, origin, 0.02, counts, 0.05)
    assert np.abs(s - direct).max() < 1e-11
