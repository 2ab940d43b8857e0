"""GPU: the engine-level spectral API (R/convolution.py:164-313) against numpy /
the oracle's restatement of the reference engine: fft_forward / fft_inverse on
mixed-radix, Bluestein (large prime factors) and long (global ping-pong)
axes; FftConvolver.kernel_hat / impulse_hat / forward_pair / product /
inverse_to_grid / inverse_pair_to_grid in the reference's padded shape; the
phi_fft kernel_hat reuse hook."""

import numpy as np
import pytest

import eikfld_oracle as orc
from conftest import rng_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu(cuda_ok):
    from paper_1112_3010_b200 import _native

    _native.lib()


CFG_TAU = 0.05


def _cfg():
    from paper_1112_3010_b200 import PrecisionConfig

    return PrecisionConfig.native64(CFG_TAU)


@pytest.mark.parametrize("shape", [(16,), (24,), (35,), (97,), (1000,), (1031,), (6144,), (10007,),
                                   (12, 10), (23, 19), (64, 34), (7, 11, 13), (16, 9, 25), (3, 257)])
def test_fft_forward_inverse_match_numpy(shape):
    from paper_1112_3010_b200.convolution import fft_forward, fft_inverse

    rng = rng_for(sum(shape))
    x = rng.standard_normal(shape)
    z = x + 1j * rng.standard_normal(shape)
    n = int(np.prod(shape))
    tol = 1e-15 * np.log2(max(n, 2)) * 8
    for a in (x, z):
        ref = np.fft.fftn(a)
        got = fft_forward(a, _cfg())
        assert got.shape == a.shape and got.dtype == np.complex128
        assert np.abs(got - ref).max() <= tol * np.abs(ref).max()
        back = fft_inverse(got, _cfg())
        assert np.abs(back - a).max() <= tol * np.abs(a).max()
        assert np.abs(fft_inverse(a, _cfg()) - np.fft.ifftn(a)).max() <= tol * np.abs(np.fft.ifftn(a)).max()


def test_reference_transform_kats():
    """tests/test_convolution.py:46-85 restated: zeros, the cosine's two bins, round trip, zero axis."""
    from paper_1112_3010_b200 import ValidationError
    from paper_1112_3010_b200.convolution import fft_forward, fft_inverse

    assert np.abs(fft_forward(np.zeros(16), _cfg())).max() == 0.0
    n = 32
    spec = np.abs(fft_forward(np.cos(2 * np.pi * 5 * np.arange(n) / n), _cfg()))
    hot = np.argsort(spec)[-2:]
    assert set(hot) == {5, n - 5} and spec[hot].min() > n / 2 - 1e-9
    assert np.delete(spec, hot).max() < 1e-12 * n
    x = rng_for(0).standard_normal(256)
    assert np.abs(fft_inverse(fft_forward(x, _cfg()), _cfg()).real - x).max() <= 1e-12 * np.abs(x).max()
    with pytest.raises(ValidationError):
        fft_forward(np.zeros((4, 0)), _cfg())


@pytest.mark.parametrize("counts", [(12, 10), (33,), (9, 8, 7)])
def test_convolver_building_blocks_match_oracle(counts):
    from paper_1112_3010_b200 import GridSpec, ScalarField
    from paper_1112_3010_b200.convolution import FftConvolver
    from paper_1112_3010_b200.distance import kernel_exp

    grid = GridSpec((0.0,) * len(counts), 0.05, counts)
    cfg = _cfg()
    k = kernel_exp(grid, cfg)
    conv = FftConvolver(grid, k.shape, cfg)
    oc = orc.Convolver(counts, k.shape)
    assert conv.pshape == oc.pshape
    assert conv.out_slice == oc.out_slice
    rng = rng_for(len(counts))
    g = rng.random(counts)
    k2 = k.values * rng.random(k.shape)
    scale = np.abs(np.fft.fftn(np.pad(k.values, [(0, p - s) for p, s in zip(oc.pshape, k.shape)]))).max()
    ka, kb = conv.forward_pair(k.values, k.shape, k2, k2.shape)
    ra, rb = oc.forward_pair(k.values, k.shape, k2, k2.shape)
    assert np.abs(ka - ra).max() <= 1e-13 * scale and np.abs(kb - rb).max() <= 1e-13 * scale
    kh = conv.kernel_hat(k)
    assert np.abs(kh - ra).max() <= 1e-13 * scale
    gh = conv.impulse_hat(ScalarField(grid, g.reshape(-1)))
    rgh = oc.impulse_hat(g)
    assert np.abs(gh - rgh).max() <= 1e-13 * np.abs(rgh).max()
    prod = conv.product(kh, gh)
    # numpy's complex multiply is (ac - bd) + (ad + bc) i; whether its SIMD loop
    # fuses the products depends on the host CPU, so the bit-exact check is
    # against the unfused real arithmetic and numpy's own product is held to 2 ulp
    want = (kh.real * gh.real - kh.imag * gh.imag) + 1j * (kh.real * gh.imag + kh.imag * gh.real)
    assert np.array_equal(prod, want)
    assert np.abs(prod - kh * gh).max() <= 4 * np.finfo(float).eps * np.abs(kh * gh).max()
    out = conv.inverse_to_grid(prod)
    ref = oc.inverse_to_grid(ra * rgh)
    assert out.shape == tuple(counts)
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
    pa, pb = conv.inverse_pair_to_grid(prod, conv.product(kb, gh))
    qa, qb = oc.inverse_pair_to_grid(ra * rgh, rb * rgh)
    assert np.abs(pa - qa).max() <= 1e-12 * np.abs(qa).max()
    assert np.abs(pb - qb).max() <= 1e-12 * np.abs(qb).max()
    # the fused convolve path and the building blocks agree
    fused = conv.convolve(k, ScalarField(grid, g.reshape(-1)))
    assert np.abs(fused - out).max() <= 1e-12 * np.abs(out).max()


def test_phi_fft_kernel_hat_hook():
    from paper_1112_3010_b200 import GridSpec, PrecisionConfig
    from paper_1112_3010_b200.convolution import FftConvolver
    from paper_1112_3010_b200.distance import kernel_exp, phi_fft, s_fft
    from paper_1112_3010_b200.workloads import random_node_sources

    grid = GridSpec((0.0, 0.0), 1.0 / 64, (64, 64))
    cfg = PrecisionConfig.native64(0.08)
    ps = random_node_sources(17, grid, 100)
    k = kernel_exp(grid, cfg)
    conv = FftConvolver(grid, k.shape, cfg)
    kh = conv.kernel_hat(k)
    a = phi_fft(ps, grid, cfg).values
    b = phi_fft(ps, grid, cfg, convolver=conv, kernel_hat=kh).values
    assert np.abs(a - b).max() <= 1e-12 * a.max()
    # a different spectrum is honoured, not ignored: twice the kernel, twice phi
    c = phi_fft(ps, grid, cfg, convolver=conv, kernel_hat=2.0 * kh).values
    assert np.abs(c - 2.0 * b).max() <= 1e-12 * c.max()
    s = s_fft(ps, grid, cfg, convolver=conv, kernel_hat=kh).values
    assert np.abs(s - (-cfg.tau * np.log(b))).max() <= 1e-12
