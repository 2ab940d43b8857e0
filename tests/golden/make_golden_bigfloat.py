"""Golden fixtures for the double-double path from the REAL reference's
big-float pipeline (`eikfld`, PrecisionConfig.bigfloat), run in this build
container:

    python tests/golden/make_golden_bigfloat.py

gmpy2 (MPFR/MPC) is not installed here, so the reference's gmpy2 calls are
served by a small mpmath-backed module placed first on sys.path (written to a
temp dir below; mpmath 1.3.0 is in the image).  It maps exactly the names the
reference uses (R/convolution.py:20-23,63-143; R/distance.py:38-45,95-101;
R/precision.py:74-76; R/grid.py:152-154): mpfr, mpc, context(precision=bits),
exp, sqrt, log, cos, sin, const_pi, is_finite.  mpmath rounds every operation
to the working precision like MPFR does (not bit-identically), which is all
the fixtures need: they are the reference's p = 200-bit answers, ~1e-55
relative, used as the truth the 106-bit double-double path is checked against.

Outputs tests/golden/bigfloat_*.npz (float64 S / gradient / Hessian and the
reference's phi rounded to float64 plus its log10).
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
BITS = 200

_SHIM = '''
import mpmath as _mp

mpfr = _mp.mpf
mpc = _mp.mpc
exp = _mp.exp
sqrt = _mp.sqrt
log = _mp.log
cos = _mp.cos
sin = _mp.sin
is_finite = _mp.isfinite


def const_pi():
    return +_mp.pi


def context(precision=53):
    return _mp.workprec(int(precision))
'''


def _import_reference():
    shim_dir = tempfile.mkdtemp(prefix="gmpy2mp_")
    with open(os.path.join(shim_dir, "gmpy2.py"), "w") as fh:
        fh.write(_SHIM)
    sys.path[:0] = [shim_dir, REF_SRC]
    from eikfld import derivatives, distance, grid, precision

    return derivatives, distance, grid, precision


def main():
    derivatives, distance, grid, precision = _import_reference()
    cases = {
        # sources near one corner: phi spans ~1e-26 of its max over the grid,
        # far below the float64 FFT's round-off floor (~1e-16 of max phi)
        "bigfloat_2d": dict(origin=(0.0, 0.0), h=1.0, counts=(20, 16), nodes=[0, 17, 34], tau=0.4, hess=True),
        # 1-D and 3-D, gradient only
        "bigfloat_1d": dict(origin=(0.0,), h=0.5, counts=(40,), nodes=[3, 4], tau=0.3, hess=False),
        "bigfloat_3d": dict(origin=(0.0, 0.0, 0.0), h=1.0, counts=(8, 7, 6), nodes=[0, 1, 43], tau=0.18,
                            hess=False),
    }
    for name, c in cases.items():
        g = grid.GridSpec(c["origin"], c["h"], c["counts"])
        ps = grid.PointSet.from_node_indices(g, np.array(c["nodes"], dtype=np.int64))
        cfg = precision.PrecisionConfig.bigfloat(c["tau"], BITS)
        phi = distance.phi_fft(ps, g, cfg).values
        import mpmath

        with mpmath.workprec(BITS):
            log10_phi = np.array([float(mpmath.log10(v)) for v in phi])
        S = distance.s_from_phi(distance.phi_fft(ps, g, cfg), cfg).values
        grad = derivatives.gradient(ps, g, cfg, method="fft")
        out = dict(counts=np.array(c["counts"]), h=c["h"], tau=c["tau"], nodes=np.array(c["nodes"]),
                   origin=np.array(c["origin"]), bits=BITS, phi=np.array([float(v) for v in phi]),
                   log10_phi=log10_phi, S=np.asarray(S, dtype=np.float64))
        for a, comp in enumerate(grad.components):
            out[f"g{a}"] = np.asarray(comp.values, dtype=np.float64)
        if c["hess"]:
            sxx, syy, sxy = derivatives.hessian_2d(ps, g, cfg, method="fft")
            out["hxx"], out["hyy"], out["hxy"] = (np.asarray(x.values, dtype=np.float64) for x in (sxx, syy, sxy))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "phi range", float(log10_phi.min()), float(log10_phi.max()))


if __name__ == "__main__":
    main()
