"""Unsigned distance S = -tau log(exp(-|x|/tau) * delta_Y) on the GPU.

Drop-in for the FFT entry points of R/distance.py (kernel_exp 22-47,
impulse_field 50-60, phi_fft 63-86, s_from_phi 89-111, s_fft 114-122).
The arithmetic runs in libeikfld_b200 (one fused pipeline: impulse DFT from
the node list, cached kernel spectrum, pruned r2c/c2r passes, -tau log phi
epilogue with underflow detection).  Same names, argument meaning and errors.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import PrecisionError, ValidationError
from .grid import ScalarField
from .precision import arithmetic, log_bound, require_native

_UNDERFLOW_MSG = (
    "{what} has non-positive entries after convolution; increase the precision bits "
    "(e.g. --precision big:512) or raise tau"
)
# the double-double path keeps float64's exponent range, so more bits cannot
# help it: only a larger tau does (this build runs big-float configs up to 106 bits)
_DD_UNDERFLOW_MSG = (
    "{what} has non-positive entries after the double-double (106-bit) convolution; its exponent "
    "range is float64's, so raise tau (bigfloat precision above 106 bits is not available in this build)"
)


def underflow_message(mode: str, what: str) -> str:
    return (_DD_UNDERFLOW_MSG if mode == "dd" else _UNDERFLOW_MSG).format(what=what)


def distinct_nodes(ps, grid) -> np.ndarray:
    """Sorted distinct snapped nodes with the reference's bounds check (R/distance.py:55-58)."""
    nodes = np.unique(np.asarray(ps.snapped_indices, dtype=np.int64))
    if nodes.size == 0:
        raise ValidationError("point-set must contain at least one point")
    if nodes[0] < 0 or nodes[-1] >= grid.num_nodes:
        raise ValidationError("snapped index out of grid bounds")
    return nodes


def _check_grid(grid):
    if not 1 <= len(grid.counts) <= 3:
        raise ValidationError("dimension must be 1, 2 or 3")


def kernel_exp(grid, cfg):
    """Sampled exp(-|offset|/tau) on [-(c-1), c-1]^D, as R/distance.py:22-47.

    Host-side sampling kept for API compatibility (tests, FftConvolver users);
    the GPU pipeline generates these samples on the device and never reads this.
    """
    from .convolution import KernelField

    tau = require_native(cfg)
    mesh = np.meshgrid(*[np.arange(-(c - 1), c) for c in grid.counts], indexing="ij")
    r2 = sum(m.astype(np.int64) ** 2 for m in mesh)
    return KernelField(grid.spacing, np.exp(-(grid.spacing * np.sqrt(r2.astype(np.float64))) / tau))


def impulse_field(ps, grid) -> ScalarField:
    """Unit impulses at the distinct snapped nodes (R/distance.py:50-60)."""
    vals = np.zeros(grid.num_nodes, dtype=np.float64)
    vals[distinct_nodes(ps, grid)] = 1.0
    return ScalarField(grid, vals)


def _run_phi_family(ps, grid, cfg, *, want_s: bool, what: str):
    mode, tau = arithmetic(cfg)
    _check_grid(grid)
    nodes = distinct_nodes(ps, grid)
    out = np.empty(grid.num_nodes, dtype=np.float64)
    if mode == "dd":  # big-float config: double-double convolution (R/convolution.py:67-143, p = 106)
        plan = _native.get_dd_plan(grid, tau, _native.FIELD_PHI | _native.FIELD_S)
        kw = {"S": out} if want_s else {"phi_hi": out}
        try:
            plan.run(nodes, check_underflow=True, **kw)
        except PrecisionError:
            raise PrecisionError(underflow_message(mode, what)) from None
        return out
    plan = _native.get_plan(grid, tau, _native.FIELD_PHI | _native.FIELD_S)
    kw = {"S": out} if want_s else {"phi": out}
    try:
        plan.run(nodes, check_underflow=True, **kw)
    except PrecisionError:
        raise PrecisionError(_UNDERFLOW_MSG.format(what=what)) from None
    return out


def _phi_from_kernel_hat(ps, grid, cfg, convolver, kernel_hat):
    """The reuse branch of R/distance.py:82-84: g_hat = impulse_hat(g), then
    inverse_to_grid(product(kernel_hat, g_hat)), on the device spectral API.
    kernel_hat is the caller's spectrum of shape FftConvolver.pshape (the
    reference's padded shape, so spectra from either package fit)."""
    from .convolution import FftConvolver, assert_positive

    require_native(cfg)
    conv = convolver if isinstance(convolver, FftConvolver) else FftConvolver(grid, getattr(
        convolver, "kshape", tuple(2 * c - 1 for c in grid.counts)), cfg)
    g_hat = conv.impulse_hat(impulse_field(ps, grid))
    values = conv.inverse_to_grid(conv.product(kernel_hat, g_hat)).reshape(-1)
    try:
        assert_positive(values, "phi")
    except PrecisionError:
        raise PrecisionError(_UNDERFLOW_MSG.format(what="phi")) from None
    return values


def phi_fft(ps, grid, cfg, convolver=None, kernel_hat=None) -> ScalarField:
    """phi = exp(-|x|/tau) * delta_Y on the grid; PrecisionError if any phi <= 0.

    Reuse hook (R/distance.py:63-86): without `kernel_hat` the exp kernel's
    spectrum is reused through the plan cache (a passed `convolver` needs no
    other state); with `convolver` and `kernel_hat` the given spectrum is
    applied through the spectral API.  For big-float configs phi comes from the
    double-double convolution and is returned rounded to float64 (the reference
    returns mpfr objects).
    """
    if convolver is not None and kernel_hat is not None:
        return ScalarField(grid, _phi_from_kernel_hat(ps, grid, cfg, convolver, kernel_hat))
    return ScalarField(grid, _run_phi_family(ps, grid, cfg, want_s=False, what="phi"))


def s_from_phi(phi: ScalarField, cfg) -> ScalarField:
    """S = -tau log(phi) for a given phi field (R/distance.py:89-111)."""
    _, tau = arithmetic(cfg)
    vals = np.asarray(phi.values, dtype=np.float64)
    if (vals <= 0).any():
        raise PrecisionError("phi <= 0: native64 underflow; rerun with --precision big:<bits>")
    return ScalarField(phi.grid, -tau * np.log(vals))


def s_fft(ps, grid, cfg, convolver=None, kernel_hat=None) -> ScalarField:
    """Composed pipeline (R/distance.py:114-122), fused on the device (the
    kernel_hat reuse branch goes through phi_fft + s_from_phi as in the reference)."""
    if convolver is not None and kernel_hat is not None:
        return s_from_phi(phi_fft(ps, grid, cfg, convolver, kernel_hat), cfg)
    return ScalarField(grid, _run_phi_family(ps, grid, cfg, want_s=True, what="phi"))


def r_exact(points, grid) -> ScalarField:
    """Exact distance to the nearest source (R/distance.py:155-168): the KD-tree
    nearest-neighbour distance at every node.  Host-side evaluation tool of the
    experiment protocols, not part of the convolution path."""
    from scipy.spatial import cKDTree

    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    if pts.shape[1] != grid.dim:
        raise ValidationError("point dimensionality does not match grid")
    dist, _ = cKDTree(pts).query(grid.node_coords(), k=1)
    return ScalarField(grid, np.asarray(dist, dtype=np.float64))


def error_bound(cfg, k: int) -> float:
    return log_bound(cfg.tau, k)


def clamp_nonnegative(field: ScalarField) -> ScalarField:
    return ScalarField(field.grid, np.maximum(field.values, 0.0), field.flagged_nodes)
