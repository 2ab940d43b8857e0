"""Run the reference package's own fp64 unit tests against the B200 build
(TEST INFRASTRUCTURE; a pytest plugin loaded with `-p reftest_support`).

`install()` makes `import eikfld.<module>` resolve to this build:

* eikfld.convolution / distance / derivatives / sign / grid / precision /
  errors are THIS package's modules (their public names, unchanged);
* names the build deliberately does not ship because they are the
  reference's own CPU oracles or test geometry are filled in from the test
  infrastructure, so the test files import:
    - distance.s_direct / s_direct_multi / r_exact, derivatives'
      method="direct" and DirectionalKernels: the O(N*K) direct sums, from
      oracle/eikfld_oracle.py (R/distance.py:133-168, R/derivatives.py:26-52,
      175-207);
    - eikfld.shapes (test geometry, R/shapes.py): the reference file itself,
      staged by tools/stage_reftests.py next to the tests (never committed);
    - gmpy2: a stub whose every use raises (only the big-float tests, which
      are deselected, touch it).

DESELECT lists the tests that are not run and why: every one needs the
reference's MPFR big-float engine above 106 bits, which this build replaces
by a double-double path up to 106 bits.  Every other test of
the four files must pass.
"""

from __future__ import annotations

import os
import sys
import types

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = os.path.join(REPO, "oracle", "_ref", "reftests")
FILES = ("test_convolution.py", "test_distance.py", "test_derivatives.py", "test_sign.py")

_BIG = "big-float arithmetic above 106 bits (MPFR engine; the build's big-float path is double-double)"
DESELECT = {
    "test_convolution.py::TestTransforms::test_roundtrip_bigfloat": _BIG,
    "test_convolution.py::TestTransforms::test_bigfloat_matches_native_at_128_bits": _BIG,
    "test_convolution.py::test_bigfloat_convolution_agrees_with_native": _BIG,
    "test_distance.py::TestKernelExp::test_deep_underflow_survives_only_in_bigfloat": _BIG,
    "test_distance.py::TestPipeline::test_k1_recovers_distance": _BIG + " (its second half, p = 192)",
    "test_distance.py::TestSDirect::test_cross_path_agreement_at_p512": _BIG,
    "test_distance.py::TestSDirect::test_dimension_independence": _BIG + " (p = 192)",
    "test_derivatives.py::TestGradient::test_fft_matches_direct_at_p512": _BIG,
    "test_derivatives.py::TestHessian::test_fft_matches_direct_at_p512": _BIG,
    "test_sign.py::TestWinding::test_fft_matches_direct_summation_p512": _BIG,
    "test_sign.py::TestDegree::test_fft_matches_direct_summation_p512": _BIG,
}


def _gmpy2_stub():
    m = types.ModuleType("gmpy2")

    def _raise(*a, **k):
        raise RuntimeError("gmpy2 is not available (big-float tests are deselected)")

    m.mpfr = m.mpc = m.exp = m.log = m.context = _raise
    m.__getattr__ = lambda name: _raise
    return m


def _clone(name, mod, extra=None):
    m = types.ModuleType(name)
    m.__dict__.update({k: v for k, v in vars(mod).items() if not k.startswith("__")})
    m.__doc__ = mod.__doc__
    m.__file__ = getattr(mod, "__file__", None)
    if extra:
        m.__dict__.update(extra)
    return m


def install():
    if "eikfld" in sys.modules and getattr(sys.modules["eikfld"], "_b200_alias", False):
        return
    for p in (REPO, os.path.join(REPO, "oracle")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import numpy as np

    import eikfld_oracle as orc
    import paper_1112_3010_b200 as P
    from paper_1112_3010_b200 import convolution, derivatives, distance, errors, experiments, grid, precision, sign

    sys.modules.setdefault("gmpy2", _gmpy2_stub())
    pkg = types.ModuleType("eikfld")
    pkg.__path__ = []
    pkg._b200_alias = True
    pkg.__dict__.update({k: v for k, v in vars(P).items() if not k.startswith("__")})

    # -- the reference's direct oracles (test infrastructure), reference signatures
    def s_direct_multi(ps, g, taus):
        return [grid.ScalarField(g, orc.s_direct(ps.points, g.origin, g.spacing, g.counts, float(t))) for t in taus]

    def s_direct(ps, g, cfg):
        return s_direct_multi(ps, g, [cfg.tau])[0]

    def r_exact(points, g):
        from scipy.spatial import cKDTree

        pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
        if pts.shape[1] != len(g.counts):
            raise errors.ValidationError("point dimensionality does not match grid")
        d, _ = cKDTree(pts).query(g.node_coords(), k=1)
        return grid.ScalarField(g, np.asarray(d, dtype=np.float64))

    class DirectionalKernels:
        def __init__(self, g):
            fa, inv = orc.directional_kernels(g.counts, g.spacing)
            self.axis_over_r, self.inv_r, self.shape = fa, inv, inv.shape

    def gradient(ps, g, cfg, method="fft"):
        if method != "direct":
            return derivatives.gradient(ps, g, cfg, method)
        nodes = ps.distinct_nodes()
        rat = orc.direct_ratios(nodes, g.origin, g.spacing, g.counts, cfg.tau)
        return grid.VectorField([grid.ScalarField(g, r, nodes) for r in rat])

    def hessian_2d(ps, g, cfg, method="fft"):
        if method != "direct":
            return derivatives.hessian_2d(ps, g, cfg, method)
        if len(g.counts) != 2:
            raise errors.ValidationError("second derivatives are implemented for 2D grids")
        nodes = ps.distinct_nodes()
        sx, sy, txx, tyy, txy = orc.direct_ratios(nodes, g.origin, g.spacing, g.counts, cfg.tau, hessian=True)
        it = 1.0 / cfg.tau
        return tuple(grid.ScalarField(g, v, nodes)
                     for v in (txx + it * sx * sx, tyy + it * sy * sy, txy + it * sx * sy))

    mods = {
        "errors": _clone("eikfld.errors", errors),
        "precision": _clone("eikfld.precision", precision),
        "grid": _clone("eikfld.grid", grid),
        "convolution": _clone("eikfld.convolution", convolution),
        "distance": _clone("eikfld.distance", distance,
                           {"s_direct": s_direct, "s_direct_multi": s_direct_multi, "r_exact": r_exact}),
        "derivatives": _clone("eikfld.derivatives", derivatives,
                              {"DirectionalKernels": DirectionalKernels, "gradient": gradient,
                               "hessian_2d": hessian_2d}),
        "sign": _clone("eikfld.sign", sign),
        "experiments": _clone("eikfld.experiments", experiments),
    }
    sys.modules["eikfld"] = pkg
    for k, m in mods.items():
        sys.modules["eikfld." + k] = m
        setattr(pkg, k, m)
    shapes_src = os.path.join(STAGE, "shapes.py")
    if os.path.exists(shapes_src):
        import importlib.util

        spec = importlib.util.spec_from_file_location("eikfld.shapes", shapes_src)
        shp = importlib.util.module_from_spec(spec)
        shp.__package__ = "eikfld"
        sys.modules["eikfld.shapes"] = shp
        spec.loader.exec_module(shp)
        pkg.shapes = shp


def pytest_load_initial_conftests(early_config, parser, args):
    install()  # before the staged conftest.py imports eikfld.grid


def pytest_configure(config):
    install()


def pytest_collection_modifyitems(config, items):
    keep, drop = [], []
    for it in items:
        key = it.nodeid.split("/")[-1]
        (drop if key in DESELECT else keep).append(it)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep
