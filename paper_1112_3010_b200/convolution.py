"""Engine-level zero-padded LINEAR convolution and transforms on the GPU.

Drop-in for the float64 engine of R/convolution.py: KernelField 30-64,
fft_forward / fft_inverse / _check_sizes 164-184, _padded_shape 205-209,
FftConvolver 212-366 (kernel_hat, impulse_hat, forward_pair,
inverse_to_grid, inverse_pair_to_grid, product, convolve, convolve_many),
fft_convolve 369-375, assert_positive 378-388.

Two device paths sit behind this module:

* `convolve` / `convolve_many` run the fused pipeline (csrc/pipeline.cu
  eik_convolve): pruned r2c -> fused column -> c2r passes over each axis
  padded to the power of two >= 2c-1, which is enough for a linear
  convolution restricted to the grid window (SURVEY.md exec. summary item 8),
  instead of next_fast_len(3c-2);
* the spectral building blocks (`fft_forward`, `kernel_hat`, `forward_pair`,
  `inverse_to_grid`, ...) hand spectra back as arrays, so they keep the
  reference's padded shape `pshape` = next_fast_len(c + k - 1) per axis and
  its layout (operands at the origin, output window at the kernel centre);
  their transforms are the mixed-radix / Bluestein device FFTs of
  csrc/spectral.cu.  Values agree with the reference's to float64 FFT noise.

Divergences: no 2^31-element cap (_check_sizes); big-float configs raise
ValidationError here (the big-float engine is the reference's CPU path; the
drop-in's S / gradient entry points run big-float configs up to 106 bits on
the double-double device path instead).
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


def next_fast_len(target: int) -> int:
    """Smallest 2^a 3^b 5^c 7^d 11^e >= target: scipy.fft.next_fast_len(target)
    for complex transforms, which R/convolution.py:209 calls."""
    n = max(1, int(target))
    while True:
        m = n
        for p in (2, 3, 5, 7, 11):
            while m % p == 0:
                m //= p
        if m == 1:
            return n
        n += 1


def _check_sizes(shape):
    """R/convolution.py:180-184 minus the 2^31-element cap (lifted on the device)."""
    if any(int(s) < 1 for s in shape):
        raise ValidationError(f"zero-length FFT axis in shape {tuple(shape)}")


def fft_forward(array, cfg) -> np.ndarray:
    """Unnormalized forward DFT over every axis of the array (R/convolution.py:164-169)."""
    require_native(cfg)
    arr = np.asarray(array)
    _check_sizes(arr.shape)
    return _native.fftn(arr, inverse=False)


def fft_inverse(array, cfg) -> np.ndarray:
    """Inverse DFT normalized by 1/N over every axis (R/convolution.py:172-177)."""
    require_native(cfg)
    arr = np.asarray(array)
    _check_sizes(arr.shape)
    return _native.fftn(arr, inverse=True)


def _padded_shape(grid, kshape, cfg) -> tuple:
    """next_fast_len(c + k - 1) per axis (R/convolution.py:205-209, float64 mode)."""
    return tuple(next_fast_len(c + k - 1) for c, k in zip(grid.counts, kshape))


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
        # spectral building blocks: the reference's padded shape and window
        self.pshape = _padded_shape(grid, self.kshape, cfg)
        center = tuple(s // 2 for s in self.kshape)
        self.out_slice = tuple(slice(c, c + n) for c, n in zip(center, grid.counts))

    # -- single transforms (R/convolution.py:244-251)

    def kernel_hat(self, kernel: KernelField) -> np.ndarray:
        self._check_kernel(kernel)
        return _native.fft_pair(self.pshape, kernel.values, kernel.shape, None, self.kshape)[0]

    def impulse_hat(self, impulses: ScalarField) -> np.ndarray:
        g = self._field(impulses).reshape(self.grid.counts)
        return _native.fft_pair(self.pshape, g, self.grid.counts, None, self.grid.counts)[0]

    # -- packed real transforms (R/convolution.py:264-307)

    def forward_pair(self, a, ashape, b, bshape):
        """FFTs of two real arrays from one complex transform."""
        a = np.asarray(a, dtype=np.float64).reshape(tuple(ashape))
        b = np.asarray(b, dtype=np.float64).reshape(tuple(bshape))
        return _native.fft_pair(self.pshape, a, a.shape, b, b.shape)

    def inverse_to_grid(self, hat) -> np.ndarray:
        """Inverse transform restricted to the grid window, real part."""
        hat = self._spectrum(hat)
        start = [s.start for s in self.out_slice]
        return _native.ifft_window(hat, None, start, self.grid.counts, False)[0]

    def inverse_pair_to_grid(self, hat_a, hat_b):
        """Two inverse transforms of real-sequence spectra in one pass."""
        start = [s.start for s in self.out_slice]
        return _native.ifft_window(self._spectrum(hat_a), self._spectrum(hat_b), start, self.grid.counts, True)

    def product(self, a_hat, b_hat) -> np.ndarray:
        return _native.cmul(a_hat, b_hat)

    def _spectrum(self, hat):
        hat = np.asarray(hat)
        if hat.dtype == object:
            raise ValidationError("the B200 build takes complex128 spectra only")
        if hat.shape != self.pshape:
            raise ValidationError(f"spectrum shape {hat.shape} != padded shape {self.pshape}")
        return hat

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
