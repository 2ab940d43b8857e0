"""GPU parity: the CUDA path (through the C ABI / drop-in API) vs the oracle.

Tolerances:
  T1  S, grad S, Hessian: |d| <= 1e-9 * max(|ref|, 1) on nodes with
      phi/phi_max >= 1e-5 (two independent fp64 FFT paths differ by
      ~tau*eps*phi_max/phi elsewhere);
  T2  on C1 the GPU is at least as close to the exact soft-min as the reference;
  T3  mu: |d| <= 1e-12, interior mask bit-exact;
  T4  the drop-in API raises PrecisionError whenever some phi <= 0.
"""

import math

import numpy as np
import pytest

import eikfld_oracle as orc
from conftest import load_golden, rng_for

pytestmark = pytest.mark.gpu

T1_RTOL = 1e-9
T1_PHI = 1e-5
T3_ATOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu(cuda_ok):
    from paper_1112_3010_b200 import _native

    _native.lib()
    yield
    _native.clear_plans()


def pkg():
    import paper_1112_3010_b200 as P
    from paper_1112_3010_b200 import convolution, derivatives, distance, engine, sign, workloads

    return P, convolution, derivatives, distance, engine, sign, workloads


def assert_t1(got, ref, phi, name=""):
    keep = phi >= T1_PHI * np.nanmax(phi)
    assert keep.any()
    err = np.abs(got[keep] - ref[keep]) / np.maximum(np.abs(ref[keep]), 1.0)
    assert err.max() <= T1_RTOL, f"{name}: max rel err {err.max():.3e} on {keep.mean():.3f} of nodes"


# ----------------------------------------------------------------- engine KATs


def test_engine_golden_and_kats():
    P, conv, _, dist, *_ = pkg()
    g = load_golden("engine_12x10.npz")
    grid = P.GridSpec((0.0, 0.0), float(g["spacing"]), tuple(g["counts"]))
    cfg = P.PrecisionConfig.native64(float(g["tau"]))
    k = dist.kernel_exp(grid, cfg)
    assert np.array_equal(k.values, g["kernel"])
    out = conv.fft_convolve(k, P.ScalarField(grid, g["dense"]), cfg).values
    assert np.abs(out - g["conv_dense"]).max() <= 1e-12 * np.abs(g["conv_dense"]).max()
    cv = conv.FftConvolver(grid, k.shape, cfg)
    many = cv.convolve_many([k, conv.KernelField(grid.spacing, g["k2"]), conv.KernelField(grid.spacing, k.values * 0.25)],
                            P.ScalarField(grid, g["impulses"]))
    for i in range(3):
        ref = g[f"many{i}"]
        assert np.abs(many[i].reshape(-1) - ref).max() < 1e-12 * np.abs(ref).max()
    # single impulse reproduces the kernel; no wrap-around (tests/test_convolution.py:98-138)
    imp = np.zeros(grid.num_nodes)
    imp[grid.multi_to_flat(([3], [7]))[0]] = 1.0
    one = conv.fft_convolve(k, P.ScalarField(grid, imp), cfg).as_grid()
    kc = k.center
    assert np.abs(one - k.values[kc[0] - 3: kc[0] - 3 + 12, kc[1] - 7: kc[1] - 7 + 10]).max() < 1e-13
    imp[:] = 0.0
    imp[0] = 1.0
    corner = conv.fft_convolve(k, P.ScalarField(grid, imp), cfg).as_grid()
    assert abs(corner[11, 9] - k.values[kc[0] + 11, kc[1] + 9]) < 1e-14


def test_engine_direct_sum_and_shift():
    P, conv, _, dist, _, _, wl = pkg()
    grid = P.GridSpec((0.0, 0.0), 1 / 64, (64, 64))
    cfg = P.PrecisionConfig.native64(0.08)
    ps = wl.random_node_sources(17, grid, 100)
    out = conv.fft_convolve(dist.kernel_exp(grid, cfg), dist.impulse_field(ps, grid), cfg).values
    nodes = grid.node_coords()
    srcs = grid.coords_of_flat(ps.distinct_nodes())
    d = np.linalg.norm(nodes[:, None, :] - srcs[None, :, :], axis=2)
    direct = np.exp(-d / cfg.tau).sum(axis=1)
    assert np.abs(out - direct).max() <= 1e-12 * direct.max()
    g1 = P.GridSpec((0.0,), 0.1, (32,))
    c1 = P.PrecisionConfig.native64(0.05)
    k1 = dist.kernel_exp(g1, c1)
    outs = []
    for j in (4, 11):
        v = np.zeros(32)
        v[j] = 1.0
        outs.append(conv.fft_convolve(k1, P.ScalarField(g1, v), c1).values)
    assert np.abs(outs[0][:25] - outs[1][7:]).max() < 1e-13


def test_engine_3d_matches_oracle():
    P, conv, *_ = pkg()
    rng = rng_for(3)
    counts = (6, 9, 7)
    grid = P.GridSpec((0.0,) * 3, 0.5, counts)
    ks = tuple(2 * c - 1 for c in counts)
    kern = rng.random(ks)
    field = rng.random(counts)
    got = conv.FftConvolver(grid, ks, P.PrecisionConfig.native64(1.0)).convolve(conv.KernelField(0.5, kern), P.ScalarField(grid, field))
    ref = orc.Convolver(counts, ks).convolve(kern, field)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


# ----------------------------------------------------------------- distance / derivatives


def test_line_known_answer():
    P, _, der, dist, *_ = pkg()
    g = load_golden("line_9.npz")
    grid = P.GridSpec((0.0,), 0.1, (9,))
    cfg = P.PrecisionConfig.native64(0.05)
    ps = P.PointSet.from_node_indices(grid, [2, 6])
    s = dist.s_fft(ps, grid, cfg).values
    assert s[4] == pytest.approx(0.2 - 0.05 * math.log(2.0), abs=1e-13)
    assert np.abs(s - g["S"]).max() < 1e-12
    sx = der.gradient(ps, grid, cfg).components[0].values
    keep = np.ones(9, bool)
    keep[[2, 6]] = False
    assert np.abs(sx - g["Sx"])[keep].max() < 1e-9


def test_field64_matches_reference():
    P, _, der, dist, *_ = pkg()
    g = load_golden("field_64.npz")
    grid = P.GridSpec((0.0, 0.0), 1.0, (64, 64))
    cfg = P.PrecisionConfig.native64(float(g["tau"]))
    ps = P.PointSet.from_node_indices(grid, g["nodes"])
    phi = dist.phi_fft(ps, grid, cfg).values
    assert_t1(dist.s_fft(ps, grid, cfg).values, g["S"], phi, "S")
    gr = der.gradient(ps, grid, cfg)
    assert_t1(gr.components[0].values, g["Sx"], phi, "Sx")
    assert_t1(gr.components[1].values, g["Sy"], phi, "Sy")
    assert set(gr.flagged_nodes) == set(g["nodes"])
    hs = der.hessian_2d(ps, grid, cfg)
    for f, name in zip(hs, ("Sxx", "Syy", "Sxy")):
        assert_t1(f.values, g[name], phi, name)


def test_c1_parity_and_accuracy():
    P, _, der, dist, *_ = pkg()
    g = load_golden("c1.npz")
    grid = P.GridSpec((0.0, 0.0), 1.0, (256, 256))
    cfg = P.PrecisionConfig.native64(0.5)
    ps = P.PointSet.from_node_indices(grid, g["nodes"])
    phi = dist.phi_fft(ps, grid, cfg).values
    s = dist.s_fft(ps, grid, cfg).values
    assert_t1(s, g["S"], phi, "S")
    gr = der.gradient(ps, grid, cfg)
    assert_t1(gr.components[0].values, g["Sx"], phi, "Sx")
    assert_t1(gr.components[1].values, g["Sy"], phi, "Sy")
    # T2: at least as accurate as the reference against the exact soft-min
    ours = np.abs(s - g["S_direct"]).max()
    theirs = np.abs(g["S"] - g["S_direct"]).max()
    assert ours <= theirs, (ours, theirs)


def test_underflow_raises_precision_error():
    P, _, der, dist, *_ = pkg()
    grid = P.GridSpec((0.0, 0.0), 0.1, (32, 32))
    ps = P.PointSet.from_node_indices(grid, [0])
    with pytest.raises(P.PrecisionError, match="precision"):
        dist.s_fft(ps, grid, P.PrecisionConfig.native64(1e-4))
    with pytest.raises(P.PrecisionError, match="precision"):
        der.gradient(ps, grid, P.PrecisionConfig.native64(1e-4))


def test_pipeline_properties():
    P, _, der, dist, _, _, wl = pkg()
    grid = P.GridSpec((0.0, 0.0), 0.05, (16, 16))
    cfg = P.PrecisionConfig.native64(0.05)
    ps = wl.random_node_sources(8, grid, 30)
    phi = dist.phi_fft(ps, grid, cfg)
    assert (phi.values > 0).all()
    assert phi.values[ps.distinct_nodes()].min() >= 1.0 - 1e-10
    cfg3 = P.PrecisionConfig.native64(0.03)
    ps = wl.random_node_sources(9, grid, 40)
    s = dist.s_fft(ps, grid, cfg3).values[ps.distinct_nodes()]
    assert (s <= 1e-12).all() and (s >= -cfg3.tau * math.log(40) - 1e-12).all()


def test_c2_full_size_unchecked_matches_reference():
    P, _, _, dist, eng, sign, wl = pkg()
    g = load_golden("c2_sub.npz")
    d = wl.c2()
    grid = d["grid"]
    dt = eng.DistanceTransform(grid, 0.5, grad=True, hess=True, sign=True)
    sn, sw = dt.sign_inputs(d["curve"])
    out = dt.run_host(d["points"].distinct_nodes(), sign_nodes=sn, sign_weights=sw)
    sel = g["sel"]
    phi_ref = g["phi"]
    s_ref = np.where(phi_ref > 0, -0.5 * np.log(np.where(phi_ref > 0, phi_ref, 1.0)), np.nan)
    assert_t1(out["S"][sel], s_ref, phi_ref, "S")
    assert_t1(out["grad"][0][sel], g["Sx"], phi_ref, "Sx")
    assert_t1(out["grad"][1][sel], g["Sy"], phi_ref, "Sy")
    for i, name in enumerate(("Sxx", "Syy", "Sxy")):
        assert_t1(out["hess"][i][sel], g[name], phi_ref, name)
    # T3: winding field and its rounding
    assert np.abs(out["mu"][sel] - g["mu"]).max() <= T3_ATOL
    assert abs(out["mu"].sum() - float(g["mu_sum"])) <= 1e-6
    flagged = np.zeros(grid.num_nodes, bool)
    flagged[g["flagged"]] = True
    ref_mask = (np.rint(g["mu"]) > 0)
    assert np.array_equal(out["mask"][sel][~flagged[sel]].astype(bool), ref_mask[~flagged[sel]])
    # T4: the reference raises on this config, so must the drop-in
    assert int(g["raised"]) == 1 and out["n_underflow"] > 0
    with pytest.raises(P.PrecisionError):
        dist.s_fft(d["points"], grid, P.PrecisionConfig.native64(0.5))


def test_c5_item_and_batch_consistency():
    P, _, _, _, eng, _, wl = pkg()
    g = load_golden("c5_item0_sub.npz")
    d = wl.c5(items=4)
    grid = d["grid"]
    dt = eng.DistanceTransform(grid, 0.5, grad=True)
    nodes = [p.distinct_nodes() for p in d["items"]]
    offs = np.cumsum([0] + [len(n) for n in nodes])
    batch = dt.run_host(np.concatenate(nodes), item_offsets=offs)
    sel = g["sel"]
    phi_ref = g["phi"]
    N = grid.num_nodes
    assert_t1(batch["grad"][0][:N][sel], g["Sx"], phi_ref, "Sx")
    assert_t1(batch["grad"][1][:N][sel], g["Sy"], phi_ref, "Sy")
    for i in range(4):
        single = dt.run_host(nodes[i])
        assert np.array_equal(single["S"], batch["S"][i * N:(i + 1) * N], equal_nan=True)
        assert np.array_equal(single["grad"][1], batch["grad"][1][i * N:(i + 1) * N], equal_nan=True)
    assert batch["n_underflow"] == int(batch["underflow"].sum()) > 0


# ----------------------------------------------------------------- sign


def test_winding_matches_reference_and_mask_bit_exact():
    P, _, _, _, _, sign, _ = pkg()
    g = load_golden("winding_128.npz")
    grid = P.GridSpec(tuple(g["origin"]), float(g["spacing"]), tuple(g["counts"]))
    mu = sign.winding_field(P.Curve2D(g["vertices"]), grid, P.PrecisionConfig.native64(1.0))
    assert np.abs(mu.values - g["mu"]).max() <= T3_ATOL
    assert np.array_equal(mu.flagged_nodes, g["flagged"])
    assert np.array_equal(sign.classify(mu, sign.WINDING_2D).values, g["mask"])


def test_winding_translation_equivariance_exact():
    P, _, _, _, _, sign, _ = pkg()
    h = 1 / 128
    ga = P.GridSpec((-0.125, -0.125), h, (33, 33))
    gb = P.GridSpec((-0.125 + 5 * h, -0.125 + 5 * h), h, (33, 33))
    th = 2 * np.pi * np.arange(64) / 64
    va = np.stack([0.09 * np.cos(th), 0.09 * np.sin(th)], axis=1)
    cfg = P.PrecisionConfig.native64(1.0)
    mu_a = sign.winding_field(P.Curve2D(va), ga, cfg)
    mu_b = sign.winding_field(P.Curve2D(va + 5 * h), gb, cfg)
    assert np.array_equal(mu_a.values, mu_b.values)


def test_volume_gradient_and_degree():
    P, _, der, dist, _, sign, _ = pkg()
    g = load_golden("vol_24.npz")
    grid = P.GridSpec(tuple(g["origin"]), float(g["spacing"]), tuple(g["counts"]))
    cfg = P.PrecisionConfig.native64(float(g["tau"]))
    ps = P.PointSet.from_node_indices(grid, g["nodes"])
    phi = dist.phi_fft(ps, grid, cfg).values
    assert_t1(dist.s_fft(ps, grid, cfg).values, g["S"], phi, "S")
    gr = der.gradient(ps, grid, cfg)
    for a, name in enumerate(("Sx", "Sy", "Sz")):
        assert_t1(gr.components[a].values, g[name], phi, name)
    surf = P.Surface3D(g["triangles"], g["centers"], g["normals"])
    mu = sign.degree_field(surf, grid, P.PrecisionConfig.native64(1.0))
    assert np.abs(mu.values - g["mu"]).max() <= T3_ATOL
    assert np.array_equal(sign.classify(mu, sign.DEGREE_3D).values, g["mask"])


def test_deterministic_bitwise():
    P, _, _, _, eng, _, wl = pkg()
    d = wl.c2(n=512, k=4096, radius=150.0)
    dt = eng.DistanceTransform(d["grid"], 0.5, grad=True, hess=True, sign=True)
    sn, sw = dt.sign_inputs(d["curve"])
    a = dt.run_host(d["points"].distinct_nodes(), sign_nodes=sn, sign_weights=sw)
    b = dt.run_host(d["points"].distinct_nodes(), sign_nodes=sn, sign_weights=sw)
    for k in ("S", "mu", "mask"):
        assert np.array_equal(a[k], b[k], equal_nan=True)
    for i in range(3):
        assert np.array_equal(a["hess"][i], b["hess"][i], equal_nan=True)


def test_unsorted_nodes_rejected():
    P, *_ = pkg()
    from paper_1112_3010_b200 import _native

    grid = P.GridSpec((0.0, 0.0), 1.0, (16, 16))
    plan = _native.get_plan(grid, 1.0, _native.FIELD_PHI | _native.FIELD_S)
    with pytest.raises(P.ValidationError):
        plan.run(np.array([5, 3], dtype=np.int64), S=np.empty(256), count=True)
