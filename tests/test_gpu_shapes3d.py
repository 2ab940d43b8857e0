"""Small and lopsided 3-D (and degenerate) grids against the oracle: the kernel
spectra are stored folded along every axis, so every padded length from 1 to
64 per axis, the Nyquist planes and the k1 mirror signs of the odd kernels
(gradient component 1, degree kernel 1) are exercised, through the fused and
the streamed schedule."""

import numpy as np
import pytest

import eikfld_oracle as orc
from conftest import rng_for

pytestmark = pytest.mark.gpu

SHAPES = [(3, 2, 5), (2, 3, 2), (7, 2, 9), (2, 8, 3), (16, 2, 2), (5, 9, 2), (4, 4, 4), (9, 16, 5), (2, 2, 2), (17, 3, 33)]


@pytest.mark.parametrize("streamed", ["0", "1"])
@pytest.mark.parametrize("counts", SHAPES)
def test_small_3d_shapes_vs_oracle(cuda_ok, counts, streamed, monkeypatch):
    from paper_1112_3010_b200 import GridSpec, _native, engine

    monkeypatch.setenv("EIK_STREAM3D", streamed)
    _native.clear_plans()
    h, tau = 0.5, 1.25
    grid = GridSpec((0.0, -1.0, 2.0), h, counts)
    N = grid.num_nodes
    rng = rng_for(sum(counts) * 3 + int(streamed))
    nodes = np.sort(rng.choice(N, max(1, N // 3), replace=False))
    snodes = np.sort(rng.choice(N, max(1, N // 4), replace=False))
    sw = rng.standard_normal((3, snodes.size))
    out = engine.DistanceTransform(grid, tau, grad=True, sign=True).run_host(nodes, sign_nodes=snodes, sign_weights=sw)
    ref = orc.run_config_unchecked(nodes, counts, h, tau)
    scale = np.abs(ref["phi"]).max()
    assert np.abs(np.exp(-out["S"] / tau) - ref["phi"]).max() <= 1e-12 * scale
    assert np.abs(out["S"] - ref["S"]).max() <= 1e-10
    for a in range(3):
        assert np.abs(out["grad"][a] - ref["grad"][a]).max() <= 1e-10, a
    mu_ref = orc.degree_from_weights(snodes, sw, h, counts)
    assert np.abs(out["mu"] - mu_ref).max() <= 1e-12 * max(1.0, np.abs(mu_ref).max())


# One long axis (padded to 1024 / 2048 / 4096 points) next to two short ones: the 3-D
# column kernels of those lengths read line-major kernel spectra (KSpec::ls) and run their
# wide configuration, the axis-1 lines kernels their 16-values-per-thread persistent one
# (csrc/kernels.cuh: TmCfg<.., WIDE>, LinesCfg16); cheap to check in full against the oracle.
LONG_SHAPES = [(300, 3, 2), (600, 2, 3), (1100, 2, 2), (2, 300, 3), (3, 600, 2), (2, 1100, 2), (260, 270, 2),
               (520, 530, 2), (1030, 12, 5), (12, 1030, 3), (3, 700, 130)]


@pytest.mark.parametrize("streamed", ["0", "1"])
@pytest.mark.parametrize("counts", LONG_SHAPES)
def test_long_axis_3d_shapes_vs_oracle(cuda_ok, counts, streamed, monkeypatch):
    from paper_1112_3010_b200 import GridSpec, _native, engine

    monkeypatch.setenv("EIK_STREAM3D", streamed)
    _native.clear_plans()
    h = 0.5
    tau = max(1.25, max(counts) * h / 20.0)  # keeps phi far above the FFT noise floor on the long axis
    grid = GridSpec((0.0, -1.0, 2.0), h, counts)
    N = grid.num_nodes
    rng = rng_for(sum(counts) * 7 + int(streamed))
    nodes = np.sort(rng.choice(N, max(1, N // 3), replace=False))
    snodes = np.sort(rng.choice(N, max(1, N // 4), replace=False))
    sw = rng.standard_normal((3, snodes.size))
    out = engine.DistanceTransform(grid, tau, grad=True, sign=True).run_host(nodes, sign_nodes=snodes, sign_weights=sw)
    ref = orc.run_config_unchecked(nodes, counts, h, tau)
    scale = np.abs(ref["phi"]).max()
    assert np.abs(np.exp(-out["S"] / tau) - ref["phi"]).max() <= 1e-12 * scale
    assert np.abs(out["S"] - ref["S"]).max() <= 1e-9
    for a in range(3):
        assert np.abs(out["grad"][a] - ref["grad"][a]).max() <= 1e-9, a
    mu_ref = orc.degree_from_weights(snodes, sw, h, counts)
    assert np.abs(out["mu"] - mu_ref).max() <= 1e-12 * max(1.0, np.abs(mu_ref).max())
