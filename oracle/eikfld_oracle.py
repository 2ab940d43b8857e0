"""CPU oracle for the FFT-convolution distance transform — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the float64 ("native64") path of
the reference package `eikfld` (R/ = /root/reference/pkg/src/eikfld).  It is
the checker the GPU path is compared against; it is never shipped or called by
the product (`paper_1112_3010_b200`).  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline / `--impl reference` legs may import it.

Every function performs the same floating-point operations in the same order
as the reference function it cites, so on identical inputs it reproduces the
reference bit for bit.  That claim is pinned by `tests/test_oracle_golden.py`
against fixtures produced by running the real reference in the build
container (`tests/golden/make_golden.py`).

The FFT arithmetic of the reference lives in a third-party dependency that is
not vendored under /root/reference: scipy.fft (pocketfft/ducc0 c2c), pinned
only as `scipy>=1.10` (R/../../pyproject.toml:12); the fixtures were made with
scipy 1.18.1 / numpy 2.3.5, which is also what this image ships.

Inputs are plain arrays (counts, spacing, origin, flat node indices) so the
oracle does not depend on either package's container types.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.fft as sfft

__all__ = [
    "kernel_exp", "directional_kernels", "ratio_kernel", "padded_shape",
    "Convolver", "impulse_values", "phi_unchecked", "s_fft", "gradient_unchecked",
    "hessian_2d_unchecked", "snap", "tangent_impulses", "flux_impulses",
    "winding_field", "degree_field", "classify", "s_direct", "direct_ratios",
    "winding_direct", "degree_direct", "hessian_factors", "OracleUnderflow",
    "run_config_unchecked", "phi_direct_mp", "degree_from_weights", "direct_local",
]


class OracleUnderflow(ArithmeticError):
    """Mirror of eikfld.errors.PrecisionError (R/errors.py:8-13)."""


# ---------------------------------------------------------------------------
# kernels (R/distance.py:22-47, R/derivatives.py:26-57, R/sign.py:90-105)


def _int_offsets(counts):
    return [np.arange(-(c - 1), c) for c in counts]


def kernel_exp(counts, spacing, tau):
    """exp(-h*sqrt(i^2+j^2[+k^2])/tau) on [-(c-1), c-1]^D (R/distance.py:33-37)."""
    mesh = np.meshgrid(*_int_offsets(counts), indexing="ij")
    r2 = sum(m.astype(np.int64) ** 2 for m in mesh)
    r = spacing * np.sqrt(r2.astype(np.float64))
    return np.exp(-r / tau)


def _float_mesh(counts, spacing):
    axes = [spacing * np.arange(-(c - 1), c, dtype=np.float64) for c in counts]
    return np.meshgrid(*axes, indexing="ij")


def directional_kernels(counts, spacing):
    """(axis_over_r list, inv_r); zero at the centre (R/derivatives.py:35-52)."""
    mesh = _float_mesh(counts, spacing)
    r = np.sqrt(sum(m * m for m in mesh))
    centre = tuple(c - 1 for c in counts)
    safe = r.copy()
    safe[centre] = 1.0
    fa = []
    for m in mesh:
        f = m / safe
        f[centre] = 0.0
        fa.append(f)
    inv = 1.0 / safe
    inv[centre] = 0.0
    return fa, inv


def hessian_factors(fa, inv_r, tau):
    """Eq. 40-42 factor list [fc, fs, t_xx, t_yy, t_xy] (R/derivatives.py:139-153)."""
    it = 1.0 / tau
    fc, fs = fa
    return [
        fc,
        fs,
        -it * fc * fc + fs * fs * inv_r,
        -it * fs * fs + fc * fc * inv_r,
        -(it + inv_r) * fc * fs,
    ]


def ratio_kernel(counts, spacing, axis, power):
    """offset_axis / |offset|^power, 0 at the centre (R/sign.py:97-105)."""
    mesh = _float_mesh(counts, spacing)
    r = np.sqrt(sum(m * m for m in mesh))
    centre = tuple(c - 1 for c in counts)
    r[centre] = 1.0
    vals = mesh[axis] / r**power
    vals[centre] = 0.0
    return vals


# ---------------------------------------------------------------------------
# convolution engine (R/convolution.py:152-157, 205-366)


def padded_shape(counts, kshape):
    """next_fast_len(c + k - 1) per axis (R/convolution.py:205-209)."""
    return tuple(sfft.next_fast_len(c + k - 1) for c, k in zip(counts, kshape))


def _reflect(arr):
    """arr at negated frequency indices (R/convolution.py:152-157)."""
    out = arr
    for ax in range(arr.ndim):
        out = np.roll(np.flip(out, axis=ax), 1, axis=ax)
    return out


class Convolver:
    """Zero-padded linear convolution over a grid (R/convolution.py:212-366)."""

    def __init__(self, counts, kshape):
        self.counts = tuple(int(c) for c in counts)
        self.kshape = tuple(int(k) for k in kshape)
        self.pshape = padded_shape(self.counts, self.kshape)
        centre = tuple(k // 2 for k in self.kshape)
        self.out_slice = tuple(slice(c, c + n) for c, n in zip(centre, self.counts))

    def forward_pair(self, a, ashape, b, bshape):
        za = np.zeros(self.pshape, dtype=np.complex128)
        za[tuple(slice(0, s) for s in ashape)] = np.asarray(a, dtype=np.float64)
        zb = np.zeros(self.pshape, dtype=np.float64)
        zb[tuple(slice(0, s) for s in bshape)] = b
        za += 1j * zb
        z = sfft.fftn(za)
        zr = _reflect(np.conj(z))
        return 0.5 * (z + zr), -0.5j * (z - zr)

    def _pad(self, values, shape):
        out = np.zeros(self.pshape, dtype=np.float64)
        out[tuple(slice(0, s) for s in shape)] = values
        return out

    def impulse_hat(self, g):
        return sfft.fftn(np.asarray(self._pad(g, self.counts), dtype=np.complex128))

    def inverse_to_grid(self, hat):
        full = sfft.ifftn(np.asarray(hat, dtype=np.complex128))
        return np.ascontiguousarray(full[self.out_slice].real)

    def inverse_pair_to_grid(self, ha, hb):
        full = sfft.ifftn(np.asarray(ha + 1j * hb, dtype=np.complex128))
        w = full[self.out_slice]
        return np.ascontiguousarray(w.real), np.ascontiguousarray(w.imag)

    def convolve(self, kernel, g):
        kh, gh = self.forward_pair(kernel, kernel.shape, g, self.counts)
        return self.inverse_to_grid(kh * gh)

    def convolve_many(self, kernels, g):
        """Pair-packed batch (R/convolution.py:325-366)."""
        hats = []
        i = 0
        gh = None
        if len(kernels) % 2 == 1:
            kh, gh = self.forward_pair(kernels[0], kernels[0].shape, g, self.counts)
            hats.append(kh)
            i = 1
        for j in range(i, len(kernels), 2):
            ha, hb = self.forward_pair(
                kernels[j], kernels[j].shape, kernels[j + 1], kernels[j + 1].shape
            )
            hats.extend([ha, hb])
        if gh is None:
            gh = self.impulse_hat(g)
        prods = [h * gh for h in hats]
        outs = []
        for j in range(0, len(prods) - 1, 2):
            outs.extend(self.inverse_pair_to_grid(prods[j], prods[j + 1]))
        if len(prods) % 2 == 1:
            outs.append(self.inverse_to_grid(prods[-1]))
        return outs


# ---------------------------------------------------------------------------
# distance / derivatives (R/distance.py:50-122, R/derivatives.py:64-172)


def impulse_values(nodes, counts):
    """Unit impulses at the distinct nodes (R/distance.py:50-60)."""
    g = np.zeros(int(np.prod(counts)), dtype=np.float64)
    g[np.unique(np.asarray(nodes, dtype=np.int64))] = 1.0
    return g.reshape(counts)


def phi_unchecked(nodes, counts, spacing, tau):
    """phi_fft without assert_positive (R/distance.py:63-86)."""
    k = kernel_exp(counts, spacing, tau)
    conv = Convolver(counts, k.shape)
    return conv.convolve(k, impulse_values(nodes, counts)).reshape(-1)


def s_fft(nodes, counts, spacing, tau):
    """S = -tau log phi, raising like R/convolution.py:378-388 and R/distance.py:104-110."""
    phi = phi_unchecked(nodes, counts, spacing, tau)
    if (phi <= 0).any():
        raise OracleUnderflow("phi has non-positive entries: precision")
    return -tau * np.log(phi)


def _ratios_unchecked(nodes, counts, spacing, tau, factor_fn):
    fa, inv_r = directional_kernels(counts, spacing)
    base = kernel_exp(counts, spacing, tau)
    kernels = [base] + [f * base for f in factor_fn(fa, inv_r)]
    conv = Convolver(counts, base.shape)
    outs = conv.convolve_many(kernels, impulse_values(nodes, counts))
    den = outs[0]
    return den.reshape(-1), [(num / den).reshape(-1) for num in outs[1:]]


def gradient_unchecked(nodes, counts, spacing, tau):
    """(den, [S_a]) of R/derivatives.py:64-79 via _fft_ratios (156-172)."""
    return _ratios_unchecked(nodes, counts, spacing, tau, lambda fa, ir: list(fa))


def hessian_2d_unchecked(nodes, counts, spacing, tau):
    """(den, sxx, syy, sxy) of R/derivatives.py:82-112."""
    den, (sx, sy, txx, tyy, txy) = _ratios_unchecked(
        nodes, counts, spacing, tau, lambda fa, ir: hessian_factors(fa, ir, tau)
    )
    it = 1.0 / tau
    return den, txx + it * sx * sx, tyy + it * sy * sy, txy + it * sx * sy


# ---------------------------------------------------------------------------
# sign (R/grid.py:257-278, R/sign.py:42-198)


def snap(points, origin, spacing, counts):
    """Nearest node, ties to the lower index; flat row-major (R/grid.py:257-278)."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    lo = np.asarray(origin, dtype=np.float64)
    hi = lo + (np.asarray(counts) - 1) * spacing
    if not np.all((pts >= lo) & (pts <= hi)):
        raise ValueError("point outside grid")
    t = (pts - lo) / spacing
    idx = np.ceil(t - 0.5).astype(np.int64)
    idx = np.clip(idx, 0, np.asarray(counts) - 1)
    return np.ravel_multi_index(tuple(idx[:, a] for a in range(len(counts))), counts)


def coords_of_flat(flat, origin, spacing, counts):
    multi = np.stack(np.unravel_index(np.asarray(flat), counts), axis=-1).astype(np.float64)
    return np.asarray(origin, dtype=np.float64) + spacing * multi


def tangent_impulses(vertices, origin, spacing, counts):
    """Snapped chord tangents scattered with np.add.at (R/sign.py:42-57)."""
    snapped_idx = snap(vertices, origin, spacing, counts)
    snapped = coords_of_flat(snapped_idx, origin, spacing, counts)
    tang = np.roll(snapped, -1, axis=0) - snapped
    n = int(np.prod(counts))
    g1 = np.zeros(n)
    g2 = np.zeros(n)
    np.add.at(g1, snapped_idx, tang[:, 0])
    np.add.at(g2, snapped_idx, tang[:, 1])
    return np.unique(snapped_idx), g1, g2


def flux_impulses(triangles, centers, normals, origin, spacing, counts):
    """Area-weighted normals at snapped centres (R/sign.py:68-86)."""
    idx = snap(centers, origin, spacing, counts)
    e1 = triangles[:, 1] - triangles[:, 0]
    e2 = triangles[:, 2] - triangles[:, 0]
    areas = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
    weighted = normals * areas[:, None]
    n = int(np.prod(counts))
    gs = []
    for a in range(3):
        g = np.zeros(n)
        np.add.at(g, idx, weighted[:, a])
        gs.append(g)
    return np.unique(idx), gs


def winding_field(vertices, origin, spacing, counts):
    """mu = (ksr*g1 - kcr*g2)/(2 pi) (R/sign.py:108-132); returns (mu, flagged)."""
    flagged, g1, g2 = tangent_impulses(vertices, origin, spacing, counts)
    kcr = ratio_kernel(counts, spacing, 0, 2)
    ksr = ratio_kernel(counts, spacing, 1, 2)
    conv = Convolver(counts, kcr.shape)
    kcr_h, ksr_h = conv.forward_pair(kcr, kcr.shape, ksr, ksr.shape)
    g1_h, g2_h = conv.forward_pair(g1.reshape(counts), counts, g2.reshape(counts), counts)
    h = ksr_h * g1_h - kcr_h * g2_h
    mu = conv.inverse_to_grid(h)
    return mu.reshape(-1) / (2.0 * math.pi), flagged


def degree_field(triangles, centers, normals, origin, spacing, counts):
    """mu = -sum_a (o_a/r^3 * g_a)/(4 pi) (R/sign.py:135-163); returns (mu, flagged)."""
    flagged, gs = flux_impulses(triangles, centers, normals, origin, spacing, counts)
    ks = [ratio_kernel(counts, spacing, a, 3) for a in range(3)]
    conv = Convolver(counts, ks[0].shape)
    k0, k1 = conv.forward_pair(ks[0], ks[0].shape, ks[1], ks[1].shape)
    k2, g0 = conv.forward_pair(ks[2], ks[2].shape, gs[0].reshape(counts), counts)
    g1, g2 = conv.forward_pair(gs[1].reshape(counts), counts, gs[2].reshape(counts), counts)
    h = k0 * g0 + k1 * g1 + k2 * g2
    mu = conv.inverse_to_grid(h)
    return -mu.reshape(-1) / (4.0 * math.pi), flagged


def degree_from_weights(nodes, weights, spacing, counts):
    """degree_field's convolution (R/sign.py:135-163) fed per-node weight vectors
    (nodes: distinct flat indices; weights: (3, len(nodes)), already summed per
    node as FluxData.build's np.add.at does) instead of triangle centres: the
    C4 workload's vertex normals.  Same kernels, packing and order."""
    n = int(np.prod(counts))
    gs = []
    for a in range(3):
        g = np.zeros(n)
        g[np.asarray(nodes, dtype=np.int64)] = weights[a]
        gs.append(g)
    ks = [ratio_kernel(counts, spacing, a, 3) for a in range(3)]
    conv = Convolver(counts, ks[0].shape)
    k0, k1 = conv.forward_pair(ks[0], ks[0].shape, ks[1], ks[1].shape)
    k2, g0 = conv.forward_pair(ks[2], ks[2].shape, gs[0].reshape(counts), counts)
    g1, g2 = conv.forward_pair(gs[1].reshape(counts), counts, gs[2].reshape(counts), counts)
    h = k0 * g0 + k1 * g1 + k2 * g2
    mu = conv.inverse_to_grid(h)
    return -mu.reshape(-1) / (4.0 * math.pi)


def degree_direct_nodes(nodes, weights, query, spacing, counts, chunk=16):
    """The degree convolution of degree_from_weights (R/sign.py:135-163) as the
    plain sums it equals, at selected query nodes (flat indices):
    mu(x) = -(1 / 4 pi) sum_v sum_a w_a(v) o_a / |o|^3, o = h (i_x - i_v), with
    the zero offset contributing nothing (R/sign.py:97-105).  O(Q K): the exact
    checker where the FFT oracle does not fit (C4 at 1024^3)."""
    nodes = np.asarray(nodes, dtype=np.int64)
    query = np.asarray(query, dtype=np.int64)
    ijk_v = np.stack(np.unravel_index(nodes, counts), axis=1).astype(np.float64)
    ijk_q = np.stack(np.unravel_index(query, counts), axis=1).astype(np.float64)
    w = np.asarray(weights, dtype=np.float64)  # (3, K)
    out = np.empty(query.size)
    for lo in range(0, query.size, chunk):
        o = spacing * (ijk_q[lo:lo + chunk, None, :] - ijk_v[None, :, :])  # (q, K, 3)
        r2 = np.einsum("qka,qka->qk", o, o)
        r3 = r2 * np.sqrt(r2)
        num = np.einsum("qka,ak->qk", o, w)
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.where(r2 > 0.0, num / r3, 0.0)
        out[lo:lo + chunk] = -t.sum(axis=1) / (4.0 * math.pi)
    return out


def direct_local(src, query, tau, hessian=False, cutoff=30.0):
    """s_direct / direct_ratios (R/distance.py:133-152, R/derivatives.py:186-207)
    at selected query points, summing only the sources within dmin + cutoff of
    each query (kd-tree).  The dropped terms carry weight exp(-cutoff/tau) or
    less relative to the nearest one (cutoff 30, tau 0.5: e^-60), far below
    float64 resolution, so this equals the full sums; it makes the exact
    checker affordable at C3 scale.  Returns (S, [ratios...])."""
    from scipy.spatial import cKDTree

    src = np.asarray(src, dtype=np.float64)
    query = np.atleast_2d(np.asarray(query, dtype=np.float64))
    tree = cKDTree(src)
    dmin, _ = tree.query(query)
    S = np.empty(query.shape[0])
    nf = (5 if hessian else src.shape[1])
    acc = [np.empty(query.shape[0]) for _ in range(nf)]
    for q in range(query.shape[0]):
        idx = tree.query_ball_point(query[q], dmin[q] + cutoff)
        diff = query[q][None, :] - src[idx]
        dist = np.sqrt(np.einsum("ij,ij->i", diff, diff))
        r = dist.min()
        w = np.exp(-(dist - r) / tau)
        den = w.sum()
        S[q] = r - tau * np.log(den)
        zero = dist == 0.0
        safe = np.where(zero, 1.0, dist)
        fa = [np.where(zero, 0.0, diff[:, a] / safe) for a in range(diff.shape[1])]
        ir = np.where(zero, 0.0, 1.0 / safe)
        facs = hessian_factors(fa, ir, tau) if hessian else fa
        for a, f in enumerate(facs):
            acc[a][q] = (f * w).sum() / den
    return S, acc


def classify(mu, flagged, counts, mode, threshold=None):
    """Interior mask with nearest-unflagged fill (R/sign.py:166-198)."""
    from scipy import ndimage

    vals = np.asarray(mu, dtype=np.float64).copy()
    if flagged is not None and len(flagged):
        fl = np.zeros(vals.size, dtype=bool)
        fl[flagged] = True
        _, nearest = ndimage.distance_transform_edt(fl.reshape(counts), return_indices=True)
        fill = vals.reshape(counts)[tuple(nearest)]
        vals = np.where(fl, fill.reshape(-1), vals)
    if threshold is not None:
        inside = vals >= threshold
    elif mode == "winding2d":
        inside = np.rint(vals) > 0
    else:
        inside = np.rint(vals) >= 1
    return inside.astype(np.float64)


# ---------------------------------------------------------------------------
# arithmetic-independent oracles (R/distance.py:125-152, R/derivatives.py:175-207,
# tests/test_sign.py:34-65)

_CHUNK = 2048


def _node_coords(origin, spacing, counts):
    axes = [origin[a] + spacing * np.arange(counts[a]) for a in range(len(counts))]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=-1)


def s_direct(points, origin, spacing, counts, tau):
    """Max-shifted log-sum-exp soft-min over the given points (R/distance.py:133-152)."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    nodes = _node_coords(origin, spacing, counts)
    out = np.empty(nodes.shape[0])
    for lo in range(0, nodes.shape[0], _CHUNK):
        hi = min(lo + _CHUNK, nodes.shape[0])
        diff = nodes[lo:hi, None, :] - pts[None, :, :]
        d = np.sqrt(np.einsum("ijk,ijk->ij", diff, diff))
        r = d.min(axis=1)
        out[lo:hi] = r - tau * np.log(np.exp(-(d - r[:, None]) / tau).sum(axis=1))
    return out


def direct_ratios(nodes_flat, origin, spacing, counts, tau, hessian=False):
    """Per-node ratios with max-shifted weights (R/derivatives.py:186-207)."""
    pts = coords_of_flat(np.unique(nodes_flat), origin, spacing, counts)
    nodes = _node_coords(origin, spacing, counts)
    acc = None
    for lo in range(0, nodes.shape[0], _CHUNK):
        hi = min(lo + _CHUNK, nodes.shape[0])
        diff = nodes[lo:hi, None, :] - pts[None, :, :]
        dist = np.sqrt(np.einsum("ijk,ijk->ij", diff, diff))
        zero = dist == 0.0
        w = np.exp(-(dist - dist.min(axis=1)[:, None]) / tau)
        safe = np.where(zero, 1.0, dist)
        fa = [np.where(zero, 0.0, diff[..., a] / safe) for a in range(diff.shape[-1])]
        ir = np.where(zero, 0.0, 1.0 / safe)
        facs = hessian_factors(fa, ir, tau) if hessian else fa
        if acc is None:
            acc = [np.empty(nodes.shape[0]) for _ in facs]
        den = w.sum(axis=1)
        for a, f in enumerate(facs):
            acc[a][lo:hi] = (f * w).sum(axis=1) / den
    return acc


def winding_direct(vertices, origin, spacing, counts):
    """Per-node discrete winding sum over snapped vertices (tests/test_sign.py:34-48)."""
    idx = snap(vertices, origin, spacing, counts)
    verts = coords_of_flat(idx, origin, spacing, counts)
    z = np.roll(verts, -1, axis=0) - verts
    nodes = _node_coords(origin, spacing, counts)
    mu = np.zeros(nodes.shape[0])
    for v, t in zip(verts, z):
        rel = v - nodes
        r2 = np.einsum("ij,ij->i", rel, rel)
        safe = np.where(r2 > 0, r2, 1.0)
        mu += np.where(r2 > 0, (rel[:, 0] * t[1] - rel[:, 1] * t[0]) / safe, 0.0)
    return mu / (2.0 * math.pi)


def degree_direct(triangles, centers, normals, origin, spacing, counts):
    """Per-node flux sum over snapped area-weighted centres (tests/test_sign.py:51-65)."""
    idx = snap(centers, origin, spacing, counts)
    cs = coords_of_flat(idx, origin, spacing, counts)
    e1 = triangles[:, 1] - triangles[:, 0]
    e2 = triangles[:, 2] - triangles[:, 0]
    w = normals * (0.5 * np.linalg.norm(np.cross(e1, e2), axis=1))[:, None]
    nodes = _node_coords(origin, spacing, counts)
    mu = np.zeros(nodes.shape[0])
    for c, wv in zip(cs, w):
        rel = c - nodes
        r = np.linalg.norm(rel, axis=1)
        safe = np.where(r > 0, r, 1.0)
        mu += np.where(r > 0, np.einsum("ij,j->i", rel, wv) / safe**3, 0.0)
    return mu / (4.0 * math.pi)


# ---------------------------------------------------------------------------
# whole-config driver used by the parity tests and the CPU baseline


def run_config_unchecked(nodes, counts, spacing, tau, want_hessian=False):
    """phi, S (NaN where phi<=0), gradient and optionally Hessian for one point set.

    Same arithmetic as s_fft + gradient(method="fft") [+ hessian_2d] minus the
    assert_positive checks, so configs whose reference call raises
    PrecisionError still have parity values on the well-conditioned nodes.
    """
    phi = phi_unchecked(nodes, counts, spacing, tau)
    with np.errstate(invalid="ignore", divide="ignore"):
        s = -tau * np.log(phi)
    s[phi <= 0] = np.nan
    den, grads = gradient_unchecked(nodes, counts, spacing, tau)
    out = {"phi": phi, "S": s, "grad_den": den, "grad": grads}
    if want_hessian:
        hden, sxx, syy, sxy = hessian_2d_unchecked(nodes, counts, spacing, tau)
        out.update(hess_den=hden, hess=[sxx, syy, sxy])
    return out


# ---------------------------------------------------------------------------
# Extended-precision checker for the double-double path


def phi_direct_mp(nodes, counts, spacing, tau, dps=60):
    """phi(x) = sum_y exp(-h |i_x - i_y| / tau) over the distinct source nodes,
    every term in mpmath at `dps` digits; returns log10(phi) per node (float64).

    The exact value the big-float FFT path of the reference approximates
    (R/distance.py:38-45 samples exp(-sqrt(q) * (h / tau)) at integer q; the
    convolution sums those samples).  Pure Python: small grids only.
    """
    import mpmath

    counts = tuple(int(c) for c in counts)
    nodes = np.asarray(nodes, dtype=np.int64)
    idx = np.stack(np.unravel_index(np.arange(int(np.prod(counts))), counts), axis=1)
    src = idx[nodes]
    out = np.empty(idx.shape[0])
    with mpmath.workdps(dps):
        scale = mpmath.mpf(spacing) / mpmath.mpf(tau)
        for n in range(idx.shape[0]):
            q = ((src - idx[n]) ** 2).sum(axis=1)
            acc = mpmath.mpf(0)
            for qq in q:
                acc += mpmath.exp(-mpmath.sqrt(int(qq)) * scale)
            out[n] = float(mpmath.log10(acc))
    return out
