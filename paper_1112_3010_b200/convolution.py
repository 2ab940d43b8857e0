"""Engine-level zero-padded LINEAR convolution on the GPU.

Drop-in for the float64 engine of R/convolution.py: KernelField 30-64,
FftConvolver 212-366 (convolve, convolve_many), fft_convolve 369-375,
assert_positive 378-388.  Arbitrary (user) kernels are transformed on the
device into full complex half-spectra; the field goes through the same
pruned r2c -> fused column -> c2r passes as the distance pipeline.

Padding differs from the reference by design: each axis is padded to the
power of two >= 2c-1 (enough for a linear convolution restricted to the grid
window; SURVEY.md exec. summary item 8) instead of next_fast_len(3c-2), and
there is no 2^31-element cap.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import PrecisionError, ValidationError
from .grid import ScalarField
from .precision import require_native


@dataclass(frozen=True)
class KernelField:
    """Kernel samples on the centred offset lattice (odd length per axis)."""

    spacing: float
    values: np.ndarray

    def __post_init__(self):
        vals = np.asarray(self.values)
        if any(s % 2 == 0 for s in vals.shape):
            raise ValidationError("kernel axes must have odd length (centered)")
        if vals.dtype == object:
            raise ValidationError("the B200 build takes float64 kernels only")
        if not np.isfinite(vals).all():
            raise ValidationError("kernel contains non-finite samples")
        object.__setattr__(self, "values", vals)

    @property
    def shape(self) -> tuple:
        return self.values.shape

    @property
    def center(self) -> tuple:
        return tuple(s // 2 for s in self.values.shape)

    def covers(self, grid) -> bool:
        return all(s >= 2 * c - 1 for s, c in zip(self.shape, grid.counts))


class FftConvolver:
    """Reusable linear-convolution plan over one grid (R/convolution.py:212-366)."""

    def __init__(self, grid, kernel_shape, cfg):
        require_native(cfg)
        self.grid = grid
        self.cfg = cfg
        self.kshape = tuple(int(k) for k in kernel_shape)
        if len(self.kshape) != len(grid.counts):
            raise ValidationError("kernel dimensionality does not match the grid")
        if any(s < 2 * c - 1 for s, c in zip(self.kshape, grid.counts)):
            raise ValidationError("kernel extent must cover the grid extent")
        if any(c < 1 for c in grid.counts):
            raise ValidationError(f"zero-length FFT axis in shape {grid.counts}")
        self.pshape = tuple(1 << max(1, int(2 * c - 1 - 1).bit_length()) for c in grid.counts)

    def _check_kernel(self, kernel: KernelField):
        if not np.isclose(kernel.spacing, self.grid.spacing, rtol=1e-12, atol=0):
            raise ValidationError(f"kernel spacing {kernel.spacing} != grid spacing {self.grid.spacing}")
        if kernel.shape != self.kshape:
            raise ValidationError("kernel shape does not match convolver plan")

    def _field(self, impulses: ScalarField):
        if impulses.grid.counts != self.grid.counts:
            raise ValidationError("impulse field lives on a different grid")
        if not np.isclose(impulses.grid.spacing, self.grid.spacing, rtol=1e-12, atol=0):
            raise ValidationError(f"kernel spacing {self.grid.spacing} != grid spacing {impulses.grid.spacing}")
        return np.asarray(impulses.values, dtype=np.float64)

    def convolve(self, kernel: KernelField, impulses: ScalarField) -> np.ndarray:
        """output(X) = sum_nodes kernel(X - node) * impulses(node), shaped like the grid."""
        self._check_kernel(kernel)
        out = _native.convolve(self.grid.counts, kernel.values[None], self._field(impulses))
        return out[0].reshape(self.grid.counts)

    def convolve_many(self, kernels, impulses: ScalarField):
        kernels = list(kernels)
        if not kernels:
            return []
        for k in kernels:
            self._check_kernel(k)
        stack = np.stack([np.asarray(k.values, dtype=np.float64) for k in kernels])
        out = _native.convolve(self.grid.counts, stack, self._field(impulses))
        return [o.reshape(self.grid.counts) for o in out]


def fft_convolve(kernel: KernelField, impulses: ScalarField, cfg) -> ScalarField:
    conv = FftConvolver(impulses.grid, kernel.shape, cfg)
    if not np.isclose(kernel.spacing, impulses.grid.spacing, rtol=1e-12, atol=0):
        raise ValidationError(f"kernel spacing {kernel.spacing} != grid spacing {impulses.grid.spacing}")
    return ScalarField(impulses.grid, conv.convolve(kernel, impulses).reshape(-1))


def assert_positive(values, what: str):
    if bool((np.asarray(values) <= 0).any()):
        raise PrecisionError(
            f"{what} has non-positive entries after convolution; increase the "
            "precision bits (e.g. --precision big:512) or raise tau"
        )
