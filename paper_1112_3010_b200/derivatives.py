"""Gradient and 2-D Hessian of S as convolution ratios, on the GPU.

Drop-in for R/derivatives.py (gradient 64-79, hessian_2d 82-112,
gradient_magnitude 115-118, level_set_curvature 121-127).  All components
come from ONE shared transform of delta_Y: the device multiplies it by the
cached spectra of exp, (o_a/|o|) exp and the Eq. 40-42 Hessian kernels and
runs one inverse per component, with the ratio/Hessian assembly fused into
the last inverse pass.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .distance import distinct_nodes, underflow_message
from .errors import PrecisionError, ValidationError
from .grid import ScalarField, VectorField
from .precision import arithmetic


def _method(method):
    if method == "fft":
        return
    if method == "direct":
        raise ValidationError(
            "method='direct' is the reference's O(N*K) CPU oracle; the B200 build provides method='fft'"
        )
    raise ValidationError(f"unknown derivative method {method!r}")


def gradient(ps, grid, cfg, method: str = "fft") -> VectorField:
    """S_a = (f_a exp * delta)/(exp * delta); flagged = distinct source nodes."""
    _method(method)
    mode, tau = arithmetic(cfg)
    nodes = distinct_nodes(ps, grid)
    fields = _native.FIELD_PHI | _native.FIELD_S | _native.FIELD_GRAD
    plan = _native.get_dd_plan(grid, tau, fields) if mode == "dd" else _native.get_plan(grid, tau, fields)
    comps = [np.empty(grid.num_nodes) for _ in range(len(grid.counts))]
    try:
        plan.run(nodes, grad=comps, check_underflow=True)
    except PrecisionError:
        raise PrecisionError(underflow_message(mode, "gradient denominator")) from None
    return VectorField([ScalarField(grid, c, nodes) for c in comps])


def hessian_2d(ps, grid, cfg, method: str = "fft"):
    """(S_xx, S_yy, S_xy): ratio term + (1/tau) S_a S_b (R/derivatives.py:82-112)."""
    if len(grid.counts) != 2:
        raise ValidationError("second derivatives are implemented for 2D grids")
    _method(method)
    mode, tau = arithmetic(cfg)
    nodes = distinct_nodes(ps, grid)
    fields = _native.FIELD_PHI | _native.FIELD_S | _native.FIELD_GRAD | _native.FIELD_HESS
    plan = _native.get_dd_plan(grid, tau, fields) if mode == "dd" else _native.get_plan(grid, tau, fields)
    h = [np.empty(grid.num_nodes) for _ in range(3)]
    try:
        plan.run(nodes, hess=h, check_underflow=True)
    except PrecisionError:
        raise PrecisionError(underflow_message(mode, "gradient denominator")) from None
    return tuple(ScalarField(grid, x, nodes) for x in h)


def gradient_magnitude(v: VectorField) -> ScalarField:
    sq = sum(np.asarray(c.values, dtype=np.float64) ** 2 for c in v.components)
    return ScalarField(v.grid, np.sqrt(sq), v.flagged_nodes)


def level_set_curvature(v: VectorField, sxx, syy, sxy) -> ScalarField:
    gx = v.components[0].values
    gy = v.components[1].values
    num = sxx.values * gy**2 - 2.0 * sxy.values * gx * gy + syy.values * gx**2
    den = np.maximum((gx**2 + gy**2) ** 1.5, 1e-300)
    return ScalarField(v.grid, num / den, v.flagged_nodes)
