"""Winding number (2-D) and topological degree (3-D) sign fields on the GPU.

Drop-in for R/sign.py (WINDING_2D/DEGREE_3D 24-25, TangentData 34-57,
FluxData 60-86, winding_field 108-132, degree_field 135-163, classify
166-198, signed_distance 201-208).  The weighted impulses are accumulated per
node on the host in exactly the order np.add.at uses (so the weights are
bit-identical to the reference's), then the device runs the same spectral
pipeline as the distance: impulse DFTs straight from the (node, weight)
lists, multiply by the cached x/r^2 (2-D) or x/r^3 (3-D) kernel spectra,
summed, one inverse, mu = h/(2 pi) or -h/(4 pi) in the fused epilogue.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ValidationError
from .grid import ScalarField, snap_points
from .precision import require_native

WINDING_2D = "winding2d"
DEGREE_3D = "degree3d"


def _accumulate(idx: np.ndarray, weights: np.ndarray):
    """Distinct nodes and per-node sums in np.add.at order (sequential, from 0.0)."""
    nodes, inv = np.unique(idx, return_inverse=True)
    acc = np.zeros((weights.shape[1], nodes.size))
    for a in range(weights.shape[1]):
        np.add.at(acc[a], inv, weights[:, a])
    return nodes, acc


def _dense(grid, nodes, values):
    g = np.zeros(grid.num_nodes)
    g[nodes] = values
    return ScalarField(grid, g)


@dataclass(frozen=True)
class TangentData:
    """Snapped chord tangents per vertex and their per-node sums (R/sign.py:34-57)."""

    vertex_nodes: np.ndarray
    tangents: np.ndarray
    nodes: np.ndarray
    weights: np.ndarray  # (2, len(nodes))
    grid: object = None

    @classmethod
    def build(cls, curve, grid) -> "TangentData":
        if len(grid.counts) != 2:
            raise ValidationError("winding numbers need a 2D grid")
        ps = snap_points(curve.vertices, grid)
        snapped = grid.coords_of_flat(ps.snapped_indices)
        tangents = np.roll(snapped, -1, axis=0) - snapped
        nodes, w = _accumulate(ps.snapped_indices, tangents)
        return cls(vertex_nodes=nodes, tangents=tangents, nodes=nodes, weights=w, grid=grid)

    # the reference's dense impulse fields (R/sign.py:36-37), built on demand
    # from the per-node sums (same values: np.add.at order)
    g1 = property(lambda self: _dense(self.grid, self.nodes, self.weights[0]))
    g2 = property(lambda self: _dense(self.grid, self.nodes, self.weights[1]))


@dataclass(frozen=True)
class FluxData:
    """Area-weighted normals at snapped triangle centres (R/sign.py:60-86)."""

    center_nodes: np.ndarray
    nodes: np.ndarray
    weights: np.ndarray  # (3, len(nodes))
    grid: object = None

    # the reference's dense impulse fields (R/sign.py:64), built on demand
    impulses = property(lambda self: tuple(_dense(self.grid, self.nodes, w) for w in self.weights))

    @classmethod
    def build(cls, surface, grid) -> "FluxData":
        if len(grid.counts) != 3:
            raise ValidationError("topological degree needs a 3D grid")
        ps = snap_points(surface.centers, grid)
        e1 = surface.triangles[:, 1] - surface.triangles[:, 0]
        e2 = surface.triangles[:, 2] - surface.triangles[:, 0]
        areas = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
        nodes, w = _accumulate(ps.snapped_indices, surface.normals * areas[:, None])
        return cls(center_nodes=nodes, nodes=nodes, weights=w, grid=grid)


def _sign_run(grid, tau, field_bit, nodes, weights, want_mask=False):
    plan = _native.get_plan(grid, tau, field_bit)
    mu = np.empty(grid.num_nodes)
    mask = np.empty(grid.num_nodes, dtype=np.uint8) if want_mask else None
    plan.run(sign_nodes=np.ascontiguousarray(nodes, dtype=np.int64),
             sign_weights=np.ascontiguousarray(weights, dtype=np.float64), mu=mu, mask=mask)
    return mu, mask


def winding_field(curve, grid, cfg) -> ScalarField:
    """Winding number at every node, counter-clockwise positive; vertex nodes flagged."""
    tau = require_native(cfg)
    data = TangentData.build(curve, grid)
    mu, _ = _sign_run(grid, tau, _native.FIELD_WINDING, data.nodes, data.weights)
    return ScalarField(grid, mu, flagged_nodes=data.vertex_nodes)


def degree_field(surface, grid, cfg) -> ScalarField:
    """Normalized flux (topological degree); triangle-centre nodes flagged."""
    tau = require_native(cfg)
    data = FluxData.build(surface, grid)
    mu, _ = _sign_run(grid, tau, _native.FIELD_DEGREE, data.nodes, data.weights)
    return ScalarField(grid, mu, flagged_nodes=data.center_nodes)


def classify(mu: ScalarField, mode: str, threshold: float | None = None) -> ScalarField:
    """Interior mask: rint(mu) > 0 (2-D) / >= 1 (3-D) or mu >= threshold.

    Flagged nodes take the value of their nearest unflagged node (grid-index
    metric) exactly as R/sign.py:166-198 does via scipy's EDT: the GPU runs the
    same separable feature transform with the same tie rules
    (csrc/classify.cu, checked against scipy in the tests).
    """
    if mode not in (WINDING_2D, DEGREE_3D):
        raise ValidationError(f"unknown classification mode {mode!r}")
    flagged = mu.flagged_nodes
    if flagged is not None and flagged.size and np.unique(flagged).size >= mu.grid.num_nodes:
        raise ValidationError("every node is flagged; cannot classify")
    mask, _ = _native.classify(mu.grid.counts, mu.values, flagged if (flagged is not None and flagged.size) else None,
                               1 if mode == WINDING_2D else 2, threshold)
    return ScalarField(mu.grid, mask, flagged_nodes=mu.flagged_nodes)


def signed_distance(s: ScalarField, mask: ScalarField) -> ScalarField:
    """Positive inside, negative outside (R/sign.py:201-208)."""
    if mask.grid != s.grid:
        raise ValidationError("mask and distance field grids differ")
    vals = np.asarray(s.values, dtype=np.float64)
    m = np.asarray(mask.values, dtype=np.float64)
    # `mask > 0.5` of the reference == `mask >= nextafter(0.5, 1)` (threshold rule)
    _, sd = _native.classify(s.grid.counts, m, None, 1, float(np.nextafter(0.5, 1.0)), S=vals)
    return ScalarField(s.grid, sd, s.flagged_nodes)


_TWO_PI = 2.0 * math.pi
