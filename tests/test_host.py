"""CPU-side tests: boundary types, host-side impulse preparation, workloads,
and that the C-ABI library loads and exports every symbol the header declares
(no compute calls — there is no GPU here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO, rng_for

import paper_1112_3010_b200 as P
from paper_1112_3010_b200 import _native, sign, workloads


def header_symbols():
    text = open(os.path.join(REPO, "include", "eikfld_b200.h")).read()
    return sorted(set(re.findall(r"\b(eik_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(_native.exported_symbols())


def test_precision_config():
    with pytest.raises(P.ValidationError):
        P.PrecisionConfig.native64(0.0)
    with pytest.raises(P.ValidationError):
        P.PrecisionConfig.bigfloat(0.1, 32)
    assert P.PrecisionConfig.parse("f64", 0.1).mode == "native64"
    assert P.PrecisionConfig.parse("big:256", 0.1).bits == 256
    with pytest.raises(P.ValidationError):
        P.PrecisionConfig.parse("quad", 0.1)


def test_bigfloat_wider_than_double_double_rejected():
    """bits <= 106 run the double-double path (GPU); wider big-float configs are
    rejected before any device work (no CPU fallback, no silent downgrade)."""
    from paper_1112_3010_b200 import derivatives, distance
    from paper_1112_3010_b200.precision import DD_BITS, arithmetic

    grid = P.GridSpec((0.0,), 0.1, (8,))
    ps = P.PointSet.from_node_indices(grid, [3])
    for fn in (distance.s_fft, distance.phi_fft, derivatives.gradient):
        with pytest.raises(P.ValidationError, match="double-double"):
            fn(ps, grid, P.PrecisionConfig.bigfloat(0.1, 128))
    assert arithmetic(P.PrecisionConfig.bigfloat(0.1, DD_BITS)) == ("dd", 0.1)
    assert arithmetic(P.PrecisionConfig.native64(0.1)) == ("f64", 0.1)


def test_grid_and_snapping():
    g = P.GridSpec((0.0, 0.0), 0.5, (4, 5))
    assert g.num_nodes == 20 and g.dim == 2
    ps = P.snap_points([[0.25, 0.25], [0.26, 1.74]], g)  # exact half goes to the lower node
    assert ps.snapped_indices[1] == 1 * 5 + 3  # t = (0.52, 3.48) -> (1, 3)
    assert ps.snapped_indices[0] == 0
    with pytest.raises(P.ValidationError):
        P.snap_points([[5.0, 0.0]], g)
    with pytest.raises(P.ValidationError):
        P.GridSpec((0.0,), 1.0, (1,))


def test_tangent_accumulation_matches_dense_add_at():
    grid = P.GridSpec((0.0, 0.0), 1.0, (64, 64))
    curve = workloads.star_curve(5, n=64, k=900, radius=18.0)
    data = sign.TangentData.build(curve, grid)
    ps = P.snap_points(curve.vertices, grid)
    snapped = grid.coords_of_flat(ps.snapped_indices)
    tang = np.roll(snapped, -1, axis=0) - snapped
    for a in range(2):
        dense = np.zeros(grid.num_nodes)
        np.add.at(dense, ps.snapped_indices, tang[:, a])
        assert np.array_equal(dense[data.nodes], data.weights[a])
    assert np.array_equal(data.vertex_nodes, np.unique(ps.snapped_indices))


def test_workload_recipes_match_survey_counts():
    assert workloads.c2()["points"].size == 5908
    assert workloads.c3()["points"].size == 105389
    assert workloads.c1()["points"].size == 2000
    v, f = workloads.icosphere(16)
    assert v.shape[0] == 10 * 16 * 16 + 2 and f.shape[0] == 20 * 16 * 16


def test_vertex_area_normals_sum_to_zero():
    v, f = workloads.perturbed_sphere(0, freq=12, radius=10.0)
    w = workloads.vertex_area_normals(v, f)
    assert np.abs(w.sum(axis=0)).max() < 1e-9
    # outward: flux of the position field equals 3 * volume > 0
    assert np.einsum("ij,ij->", v, w) > 0


def test_percentage_error_and_r_exact_match_reference_definitions():
    """metrics.percentage_error (R/metrics.py:46-72) and distance.r_exact
    (R/distance.py:155-168) against their definitions written out."""
    from paper_1112_3010_b200 import GridSpec, ScalarField
    from paper_1112_3010_b200.distance import r_exact
    from paper_1112_3010_b200.metrics import Report, percentage_error

    grid = GridSpec((0.0, -1.0), 0.5, (7, 9))
    rng = np.random.default_rng(4)
    pts = grid.node_coords()[rng.choice(grid.num_nodes, 6, replace=False)]
    ex = r_exact(pts, grid)
    brute = np.sqrt(((grid.node_coords()[:, None, :] - pts[None, :, :]) ** 2).sum(-1)).min(1)
    assert np.array_equal(ex.values, brute)
    comp = ScalarField(grid, ex.values * (1.0 + 0.01 * rng.standard_normal(grid.num_nodes)))
    st = percentage_error(comp, ex)
    inc = brute > 0
    per = 100.0 * np.abs(comp.values - brute)[inc] / brute[inc]
    assert st.included == int(inc.sum()) == grid.num_nodes - 6 and st.total == grid.num_nodes
    assert st.mean == per.mean() and st.maximum == per.max() and st.paper_mean == per.sum() / grid.num_nodes
    assert '"experiment": "x"' in Report("x", {"a": 1}, [{"b": 2}]).to_json()
