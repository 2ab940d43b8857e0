"""Generate golden fixtures by running the REAL reference package (`eikfld`).

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference imports gmpy2 at module top level (R/convolution.py:20-23,
R/precision.py:14) but its float64 path never calls it; gmpy2 is not
installed here, so a stub module whose every attribute raises is placed first
on sys.path.  Any accidental bigfloat use fails loudly.

Outputs `tests/golden/*.npz`.  These fixtures pin the numpy oracle
(`oracle/eikfld_oracle.py`) to the reference bit for bit, and the GPU parity
tests compare against the oracle/fixtures.  Large fields are stored on a
seeded node subsample plus the full-field sum so fixtures stay small.
"""

from __future__ import annotations

import math
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"

_STUB = '''
def _nope(*a, **k):
    raise RuntimeError("gmpy2 stub: bigfloat arithmetic is unavailable here")
mpc = mpfr = context = _nope
def __getattr__(name):
    return _nope
'''


def _import_reference():
    stub_dir = tempfile.mkdtemp(prefix="gmpy2stub_")
    with open(os.path.join(stub_dir, "gmpy2.py"), "w") as fh:
        fh.write(_STUB)
    sys.path[:0] = [stub_dir, REF_SRC]
    import eikfld  # noqa: F401
    from eikfld import convolution, derivatives, distance, grid, precision, sign

    return convolution, derivatives, distance, grid, precision, sign


def _subsample(n, count, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.sort(rng.choice(n, size=min(count, n), replace=False))


def make_fieldio():
    """EIKFLD01 bytes written by the reference writer (R/fieldio.py:31-64)."""
    _import_reference()
    from eikfld import fieldio, grid as grd, precision as prec

    g = grd.GridSpec(origin=(-0.5, 0.25, 1.0), spacing=0.125, counts=(4, 5, 6))
    vals = np.random.Generator(np.random.PCG64(8)).standard_normal(g.num_nodes)
    f = grd.ScalarField(g, vals, flagged_nodes=[3, 77])
    fieldio.write_field(os.path.join(HERE, "ref_field.fld"), f, "S", prec.PrecisionConfig.native64(0.1),
                        {"method": "fft", "k": 1})
    print("wrote ref_field.fld")


def main():
    if "--only-fieldio" in sys.argv:
        return make_fieldio()
    conv, der, dist, grd, prec, sgn = _import_reference()
    sys.path.insert(0, REPO)
    from paper_1112_3010_b200 import workloads as wl

    f64 = prec.PrecisionConfig.native64
    out_files = {}

    # 1. engine KATs on a small odd-shaped grid (tests/test_convolution.py:88-180)
    g = grd.GridSpec((0.0, 0.0), 0.05, (12, 10))
    cfg = f64(0.05)
    k = dist.kernel_exp(g, cfg)
    rng = np.random.Generator(np.random.PCG64(5))
    dense = rng.random(g.num_nodes)
    imp = np.zeros(g.num_nodes)
    imp[[5, 17, 80]] = 1.0
    k2 = k.values * np.random.Generator(np.random.PCG64(9)).random(k.shape)
    cv = conv.FftConvolver(g, k.shape, cfg)
    many = cv.convolve_many(
        [k, conv.KernelField(g.spacing, k2), conv.KernelField(g.spacing, k.values * 0.25)],
        grd.ScalarField(g, imp),
    )
    out_files["engine_12x10.npz"] = dict(
        counts=np.array(g.counts), spacing=g.spacing, tau=cfg.tau,
        kernel=k.values, dense=dense, impulses=imp, k2=k2,
        conv_dense=conv.fft_convolve(k, grd.ScalarField(g, dense), cfg).values,
        many0=many[0].reshape(-1), many1=many[1].reshape(-1), many2=many[2].reshape(-1),
    )

    # 2. 1D pipeline (tests/test_distance.py:91-97 style) and a 1D gradient
    g1 = grd.GridSpec((0.0,), 0.1, (9,))
    ps1 = grd.PointSet.from_node_indices(g1, [2, 6])
    c1d = f64(0.05)
    out_files["line_9.npz"] = dict(
        counts=np.array(g1.counts), spacing=g1.spacing, tau=c1d.tau, nodes=ps1.snapped_indices,
        S=dist.s_fft(ps1, g1, c1d).values,
        Sx=der.gradient(ps1, g1, c1d).components[0].values,
    )

    # 3. 2D S, gradient, Hessian on 64^2 (h=1, tau=2: no underflow)
    g64 = grd.GridSpec((0.0, 0.0), 1.0, (64, 64))
    ps = wl.random_node_sources(31, wl.GridSpec(g64.origin, g64.spacing, g64.counts), 25)
    ps = grd.PointSet.from_node_indices(g64, ps.snapped_indices)
    c64 = f64(2.0)
    gr = der.gradient(ps, g64, c64)
    hs = der.hessian_2d(ps, g64, c64)
    out_files["field_64.npz"] = dict(
        counts=np.array(g64.counts), spacing=g64.spacing, tau=c64.tau, nodes=ps.snapped_indices,
        S=dist.s_fft(ps, g64, c64).values,
        Sx=gr.components[0].values, Sy=gr.components[1].values,
        Sxx=hs[0].values, Syy=hs[1].values, Sxy=hs[2].values,
        S_direct=dist.s_direct(ps, g64, c64).values,
    )

    # 4. 2D winding on a 128^2 star curve (C2 recipe scaled), tau irrelevant for mu
    d = wl.c2(seed=3, n=128, k=1024, radius=37.5, tau=1.0)
    g128 = grd.GridSpec(d["grid"].origin, d["grid"].spacing, d["grid"].counts)
    curve = grd.Curve2D(d["curve"].vertices)
    mu = sgn.winding_field(curve, g128, f64(1.0))
    mask = sgn.classify(mu, sgn.WINDING_2D)
    out_files["winding_128.npz"] = dict(
        counts=np.array(g128.counts), spacing=g128.spacing, origin=np.array(g128.origin),
        vertices=curve.vertices, mu=mu.values, flagged=mu.flagged_nodes, mask=mask.values,
    )

    # 5. 3D gradient on 24^3 and degree of a small sphere mesh
    g3 = grd.GridSpec((-11.5,) * 3, 1.0, (24, 24, 24))
    rng = np.random.Generator(np.random.PCG64(7))
    idx3 = np.sort(rng.choice(g3.num_nodes, 60, replace=False))
    ps3 = grd.PointSet.from_node_indices(g3, idx3)
    c3d = f64(1.5)
    gr3 = der.gradient(ps3, g3, c3d)
    v, f = wl.icosphere(4)
    mesh = grd.triangulate_and_orient(v * 7.3, f)
    deg = sgn.degree_field(mesh, g3, f64(1.0))
    out_files["vol_24.npz"] = dict(
        counts=np.array(g3.counts), spacing=g3.spacing, origin=np.array(g3.origin), tau=c3d.tau,
        nodes=idx3, S=dist.s_fft(ps3, g3, c3d).values,
        Sx=gr3.components[0].values, Sy=gr3.components[1].values, Sz=gr3.components[2].values,
        triangles=mesh.triangles, centers=mesh.centers, normals=mesh.normals,
        mu=deg.values, flagged=deg.flagged_nodes,
        mask=sgn.classify(deg, sgn.DEGREE_3D).values,
    )

    # 6. C1 full size (succeeds in the reference): S, gradient, exact soft-min
    d = wl.c1()
    gC1 = grd.GridSpec(d["grid"].origin, d["grid"].spacing, d["grid"].counts)
    psC1 = grd.PointSet.from_node_indices(gC1, d["points"].snapped_indices)
    cC1 = f64(d["tau"])
    grC1 = der.gradient(psC1, gC1, cC1)
    out_files["c1.npz"] = dict(
        counts=np.array(gC1.counts), spacing=1.0, tau=cC1.tau, nodes=psC1.snapped_indices,
        S=dist.s_fft(psC1, gC1, cC1).values,
        Sx=grC1.components[0].values, Sy=grC1.components[1].values,
        S_direct=dist.s_direct(psC1, gC1, cC1).values,
    )

    # 7. C2 at full size: the public calls raise PrecisionError (T4); the
    #    unchecked FftConvolver path gives parity values.
    d = wl.c2()
    gC2 = grd.GridSpec(d["grid"].origin, d["grid"].spacing, d["grid"].counts)
    psC2 = grd.PointSet.from_node_indices(gC2, d["points"].snapped_indices)
    cC2 = f64(d["tau"])
    raised = 0
    try:
        dist.s_fft(psC2, gC2, cC2)
    except Exception as exc:  # PrecisionError
        raised = int(type(exc).__name__ == "PrecisionError")
    base = dist.kernel_exp(gC2, cC2)
    dk = der.DirectionalKernels(gC2)
    kern = [base] + [der._scaled_kernel(base, fac) for fac in der._hessian_factors(cC2.tau)(dk)]
    cvC2 = conv.FftConvolver(gC2, base.shape, cC2)
    gimp = dist.impulse_field(psC2, gC2)
    phi = cvC2.convolve(base, gimp)
    outs = cvC2.convolve_many(kern, gimp)
    den = outs[0]
    sx, sy, txx, tyy, txy = (o / den for o in outs[1:])
    it = 1.0 / cC2.tau
    muC2 = sgn.winding_field(grd.Curve2D(d["curve"].vertices), gC2, cC2)
    sel = _subsample(gC2.num_nodes, 16384, 123)
    out_files["c2_sub.npz"] = dict(
        raised=raised, sel=sel, nodes=psC2.snapped_indices, vertices=d["curve"].vertices,
        phi=phi.reshape(-1)[sel], den=den.reshape(-1)[sel],
        Sx=sx.reshape(-1)[sel], Sy=sy.reshape(-1)[sel],
        Sxx=(txx + it * sx * sx).reshape(-1)[sel], Syy=(tyy + it * sy * sy).reshape(-1)[sel],
        Sxy=(txy + it * sx * sy).reshape(-1)[sel],
        mu=muC2.values[sel], mu_sum=muC2.values.sum(), flagged=muC2.flagged_nodes,
        phi_le0=int((phi <= 0).sum()),
    )

    # 8. C5 item 0 (raises in the reference); unchecked S/gradient subsample
    d = wl.c5(items=1)
    gC5 = grd.GridSpec(d["grid"].origin, d["grid"].spacing, d["grid"].counts)
    psC5 = grd.PointSet.from_node_indices(gC5, d["items"][0].snapped_indices)
    cC5 = f64(0.5)
    base = dist.kernel_exp(gC5, cC5)
    dk = der.DirectionalKernels(gC5)
    cv5 = conv.FftConvolver(gC5, base.shape, cC5)
    g5 = dist.impulse_field(psC5, gC5)
    phi5 = cv5.convolve(base, g5)
    o5 = cv5.convolve_many([base] + [der._scaled_kernel(base, fa) for fa in dk.axis_over_r], g5)
    sel5 = _subsample(gC5.num_nodes, 16384, 321)
    out_files["c5_item0_sub.npz"] = dict(
        sel=sel5, nodes=psC5.snapped_indices, phi=phi5.reshape(-1)[sel5],
        den=o5[0].reshape(-1)[sel5],
        Sx=(o5[1] / o5[0]).reshape(-1)[sel5], Sy=(o5[2] / o5[0]).reshape(-1)[sel5],
        phi_le0=int((phi5 <= 0).sum()),
    )

    for name, arrays in out_files.items():
        path = os.path.join(HERE, name)
        np.savez_compressed(path, **arrays)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
