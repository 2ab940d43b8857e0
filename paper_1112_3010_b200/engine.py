"""Unchecked, batched, device-resident entry points (the benchmark API).

The drop-in functions (distance.s_fft, derivatives.gradient, ...) mirror the
reference: host arrays in and out, PrecisionError on any phi <= 0.  This
module is the throughput-oriented face of the same pipeline: one plan per
(grid, tau, field set), inputs/outputs may stay in HBM (torch CUDA tensors),
and underflow is reported as a per-node mask plus a count instead of an
exception — exactly the "unchecked" parity path the SURVEY prescribes for
configs whose reference call raises (SURVEY.md §7 "Underflow semantics").
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ValidationError
from .precision import require_native
from .sign import FluxData, TangentData


def field_bits(dim, want_grad=True, want_hess=False, want_sign=False):
    bits = _native.FIELD_PHI | _native.FIELD_S
    if want_grad:
        bits |= _native.FIELD_GRAD
    if want_hess:
        if dim != 2:
            raise ValidationError("second derivatives are implemented for 2D grids")
        bits |= _native.FIELD_HESS
    if want_sign:
        bits |= _native.FIELD_WINDING if dim == 2 else _native.FIELD_DEGREE
    return bits


class DistanceTransform:
    """S, grad S, Hessian (2-D) and the sign field of one grid, reusing one plan."""

    def __init__(self, grid, cfg_or_tau, *, grad=True, hess=False, sign=False, device=0):
        tau = cfg_or_tau if isinstance(cfg_or_tau, (int, float)) else require_native(cfg_or_tau)
        self.grid = grid
        self.tau = float(tau)
        self.dim = len(grid.counts)
        self.want_grad, self.want_hess, self.want_sign = grad, hess, sign
        self.plan = _native.Plan(self.dim, grid.counts, grid.spacing, self.tau,
                                 field_bits(self.dim, grad, hess, sign), device)
        self.N = int(np.prod(grid.counts))

    def sign_inputs(self, geometry):
        """(nodes, weights) for a Curve2D (2-D) or Surface3D (3-D), np.add.at order."""
        data = TangentData.build(geometry, self.grid) if self.dim == 2 else FluxData.build(geometry, self.grid)
        return data.nodes, np.ascontiguousarray(data.weights)

    def run_host(self, nodes, item_offsets=None, sign_nodes=None, sign_weights=None):
        """Host arrays in, dict of host arrays out (unchecked)."""
        B = 1 if item_offsets is None else len(item_offsets) - 1
        n = self.N * B
        out = {"S": np.empty(n), "underflow": np.empty(n, dtype=np.uint8)}
        if self.want_grad:
            out["grad"] = [np.empty(n) for _ in range(self.dim)]
        if self.want_hess:
            out["hess"] = [np.empty(n) for _ in range(3)]
        if self.want_sign and sign_nodes is not None:
            out["mu"] = np.empty(n)
            out["mask"] = np.empty(n, dtype=np.uint8)
        cnt = self.plan.run(
            np.ascontiguousarray(nodes, dtype=np.int64),
            None if item_offsets is None else np.ascontiguousarray(item_offsets, dtype=np.int64), B,
            None if sign_nodes is None else np.ascontiguousarray(sign_nodes, dtype=np.int64),
            None if sign_weights is None else np.ascontiguousarray(sign_weights, dtype=np.float64),
            S=out["S"], grad=out.get("grad", (None,) * 3), hess=out.get("hess", (None,) * 3),
            mu=out.get("mu"), mask=out.get("mask"), underflow=out["underflow"], count=True, host=True)
        out["n_underflow"] = cnt
        return out


class TauSweep:
    """S for several tau values from ONE transform of delta_Y.

    The GPU analogue of the kernel reuse in R/experiments.py:74-109 (one
    FftConvolver shared by the nine tau values of the Example-1 protocol):
    here the impulse DFT and forward column FFT are shared, each tau adds one
    cached exp spectrum, one inverse and its own -tau log phi epilogue.  3-D
    grids share the planes pass (impulse DFT along axis 2, FFT along axis 1)
    and run the axis-0 pass in chunks of four tau values.
    Unchecked: S is NaN where phi <= 0 and the total count is returned.
    """

    def __init__(self, grid, taus, device=0):
        self.grid = grid
        self.taus = [float(t) for t in taus]
        self.plan = _native.SweepPlan(len(grid.counts), grid.counts, grid.spacing, self.taus, device)

    def run_host(self, nodes):
        N = int(np.prod(self.grid.counts))
        outs = [np.empty(N) for _ in self.taus]
        n_uf = self.plan.run_sweep(np.ascontiguousarray(nodes, dtype=np.int64), outs, host=True)
        return outs, n_uf
