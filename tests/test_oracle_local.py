"""The kd-tree cut-off direct sums (oracle.direct_local, the exact checker the
C3 parity test uses) equal the oracle's full direct sums (s_direct /
direct_ratios, R/distance.py:133-152, R/derivatives.py:186-207); the
vertex-weight degree convolution equals degree_field on the same impulses."""

import numpy as np

import eikfld_oracle as orc
from conftest import load_golden, rng_for


def test_direct_local_equals_full_direct_sums():
    counts, tau = (48, 40), 0.5
    nodes = np.sort(rng_for(3).choice(48 * 40, 150, replace=False))
    src = orc.coords_of_flat(nodes, (0.0, 0.0), 1.0, counts)
    full_s = orc.s_direct(src, (0.0, 0.0), 1.0, counts, tau)
    full_h = orc.direct_ratios(nodes, (0.0, 0.0), 1.0, counts, tau, hessian=True)
    q = orc._node_coords((0.0, 0.0), 1.0, counts)
    s, h = orc.direct_local(src, q, tau, hessian=True)
    assert np.abs(s - full_s).max() <= 1e-13
    for a in range(5):
        assert np.abs(h[a] - full_h[a]).max() <= 1e-13


def test_direct_local_3d_gradient():
    counts, tau = (14, 12, 10), 0.5
    nodes = np.sort(rng_for(4).choice(14 * 12 * 10, 60, replace=False))
    src = orc.coords_of_flat(nodes, (0.0,) * 3, 1.0, counts)
    full = orc.direct_ratios(nodes, (0.0,) * 3, 1.0, counts, tau)
    s, g = orc.direct_local(src, orc._node_coords((0.0,) * 3, 1.0, counts), tau)
    assert np.abs(s - orc.s_direct(src, (0.0,) * 3, 1.0, counts, tau)).max() <= 1e-13
    for a in range(3):
        assert np.abs(g[a] - full[a]).max() <= 1e-13


def test_degree_from_weights_equals_degree_field():
    g = load_golden("vol_24.npz")
    counts = tuple(int(c) for c in g["counts"])
    origin, h = tuple(g["origin"]), float(g["spacing"])
    mu, flagged = orc.degree_field(g["triangles"], g["centers"], g["normals"], origin, h, counts)
    nodes, gs = orc.flux_impulses(g["triangles"], g["centers"], g["normals"], origin, h, counts)
    w = np.stack([gg[nodes] for gg in gs])
    assert np.array_equal(orc.degree_from_weights(nodes, w, h, counts), mu)
