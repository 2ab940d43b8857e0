"""Seeded synthetic inputs for the BASELINE.json configurations C1-C5.

The reference measures no public dataset for this path; these generators are
the fixed recipes of SURVEY.md §8(d).  All randomness is
numpy Generator(PCG64(seed)) as in R/../tests/conftest.py:7-15 and
R/experiments.py:47-48.  Shapes, sizes and value distributions follow the
config text of BASELINE.json; where the text is silent the choice is recorded
here and in DESIGN.md.
"""

from __future__ import annotations

import math

import numpy as np

from .grid import Curve2D, GridSpec, PointSet, Surface3D, snap_points


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def random_node_sources(seed: int, grid: GridSpec, k: int) -> PointSet:
    """k distinct nodes, choice(N, k, replace=False) sorted (tests/conftest.py:11-15)."""
    idx = rng_for(seed).choice(grid.num_nodes, size=k, replace=False)
    return PointSet.from_node_indices(grid, np.sort(idx))


# -- C1: 256^2, K=2000 random nodes, tau 0.5 ---------------------------------

def c1(seed: int = 0, n: int = 256, k: int = 2000):
    grid = GridSpec((0.0, 0.0), 1.0, (n, n))
    return {"grid": grid, "tau": 0.5, "points": random_node_sources(seed, grid, k)}


# -- C2: 2048^2 star curve, 16384 vertices, tau 0.5 ---------------------------

def star_curve(seed: int, n: int = 2048, k: int = 16384, radius: float = 600.0) -> Curve2D:
    """r = R(1 + .25 sin(5t+a) + .1 cos(3t+b)) centred in the grid, CCW."""
    rng = rng_for(seed)
    a, b = rng.uniform(0.0, 2.0 * math.pi, 2)
    theta = 2.0 * math.pi * np.arange(k) / k
    r = radius * (1.0 + 0.25 * np.sin(5.0 * theta + a) + 0.1 * np.cos(3.0 * theta + b))
    c = (n - 1) / 2.0
    return Curve2D(np.stack([c + r * np.cos(theta), c + r * np.sin(theta)], axis=1))


def c2(seed: int = 0, n: int = 2048, k: int = 16384, radius: float = 600.0, tau: float = 0.5):
    grid = GridSpec((0.0, 0.0), 1.0, (n, n))
    curve = star_curve(seed, n, k, radius)
    ps = PointSet.from_node_indices(grid, snap_points(curve.vertices, grid).distinct_nodes())
    return {"grid": grid, "tau": tau, "curve": curve, "points": ps}


# -- C3: 256^3, 16 random ellipsoids x 12500 surface points, tau 0.5 ----------

def ellipsoid_points(seed: int, n: int = 256, count: int = 16, per: int = 12500):
    from scipy.spatial.transform import Rotation

    rng = rng_for(seed)
    lo, hi = n / 4.0, 3.0 * n / 4.0
    pts = []
    for _ in range(count):
        centre = rng.uniform(lo, hi, 3)
        axes = rng.uniform(10.0, 40.0, 3) * (n / 256.0)
        rot = Rotation.random(random_state=rng).as_matrix()
        d = rng.standard_normal((per, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pts.append((d * axes) @ rot.T + centre)
    return np.clip(np.concatenate(pts), 0.0, n - 1.0)


def c3(seed: int = 0, n: int = 256, count: int = 16, per: int = 12500):
    grid = GridSpec((0.0, 0.0, 0.0), 1.0, (n, n, n))
    pts = ellipsoid_points(seed, n, count, per)
    ps = PointSet.from_node_indices(grid, snap_points(pts, grid).distinct_nodes())
    return {"grid": grid, "tau": 0.5, "points": ps}


# -- C4: 1024^3 perturbed icosphere, tau 0.75 ---------------------------------

def icosphere(freq: int):
    """Geodesic (class I) icosphere of frequency `freq`: V = 10 f^2 + 2 unit vertices."""
    p = (1.0 + math.sqrt(5.0)) / 2.0
    base = np.array([[-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0],
                     [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
                     [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1]], dtype=np.float64)
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    f = freq
    ii, jj = np.meshgrid(np.arange(f + 1), np.arange(f + 1), indexing="ij")
    keep = ii + jj <= f
    ii, jj = ii[keep], jj[keep]
    local = {(int(i), int(j)): n for n, (i, j) in enumerate(zip(ii, jj))}
    tri_local = []
    for i in range(f):
        for j in range(f - i):
            tri_local.append((local[i, j], local[i + 1, j], local[i, j + 1]))
            if i + j + 1 < f:
                tri_local.append((local[i + 1, j], local[i + 1, j + 1], local[i, j + 1]))
    tri_local = np.asarray(tri_local)
    verts, tris = [], []
    for n_face, (a, b, c) in enumerate(faces):
        A, B, C = base[a], base[b], base[c]
        verts.append(A + (ii[:, None] / f) * (B - A) + (jj[:, None] / f) * (C - A))
        tris.append(tri_local + n_face * len(ii))
    verts = np.concatenate(verts)
    tris = np.concatenate(tris)
    verts /= np.linalg.norm(verts, axis=1, keepdims=True)
    # merge the duplicated edge/corner vertices of neighbouring base faces
    key = np.round(verts * (8.0 * f)).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    return verts[first], inv.reshape(-1)[tris]


def _real_sph_harm(lmax, theta, phi):
    """Real orthonormal spherical harmonics Y_lm, l=1..lmax (theta polar, phi azimuth)."""
    from scipy.special import sph_harm_y

    out = []
    for l in range(1, lmax + 1):
        for m in range(-l, l + 1):
            y = sph_harm_y(l, abs(m), theta, phi)
            if m < 0:
                out.append(math.sqrt(2.0) * (-1) ** m * y.imag)
            elif m == 0:
                out.append(y.real)
            else:
                out.append(math.sqrt(2.0) * (-1) ** m * y.real)
    return np.stack(out, axis=0)


def perturbed_sphere(seed: int, freq: int = 224, radius: float = 350.0, lmax: int = 6, sigma: float = 0.05):
    """Icosphere vertices moved radially by 1 + sum_{l=1..6} c_lm Y_lm, c ~ N(0, sigma^2)."""
    v, f = icosphere(freq)
    rng = rng_for(seed)
    theta = np.arccos(np.clip(v[:, 2], -1.0, 1.0))
    phi = np.arctan2(v[:, 1], v[:, 0])
    y = _real_sph_harm(lmax, theta, phi)
    coef = rng.normal(0.0, sigma, y.shape[0])
    return v * (radius * (1.0 + coef @ y))[:, None], f


def vertex_area_normals(verts, faces):
    """Vector area per vertex: (1/3) sum over adjacent triangles of area * unit normal."""
    a, b, c = verts[faces[:, 0]], verts[faces[:, 1]], verts[faces[:, 2]]
    cross = 0.5 * np.cross(b - a, c - a)
    centre = (a + b + c) / 3.0
    flip = np.einsum("ij,ij->i", centre, cross) < 0
    cross[flip] *= -1.0
    out = np.zeros_like(verts)
    for k in range(3):
        np.add.at(out, faces[:, k], cross / 3.0)
    return out


def c4(seed: int = 0, n: int = 1024, freq: int | None = None, radius: float | None = None):
    """Perturbed icosphere in an origin-centred n^3 grid; at n = 1024: radius 350,
    frequency 224 (501,762 vertices).  Smaller n scales radius and frequency."""
    freq = freq if freq is not None else max(4, round(224 * n / 1024))
    radius = radius if radius is not None else 350.0 * n / 1024
    grid = GridSpec((-(n - 1) / 2.0,) * 3, 1.0, (n, n, n))
    v, f = perturbed_sphere(seed, freq, radius)
    w = vertex_area_normals(v, f)
    idx = snap_points(v, grid).snapped_indices
    nodes, inv = np.unique(idx, return_inverse=True)
    acc = np.zeros((3, nodes.size))
    for a in range(3):
        np.add.at(acc[a], inv, w[:, a])
    return {"grid": grid, "tau": 0.75, "vertices": v, "faces": f, "weights": w,
            "nodes": nodes, "sign_nodes": nodes, "sign_weights": acc}


def surface_from_mesh(v, f) -> Surface3D:
    from .grid import triangulate_and_orient

    return triangulate_and_orient(v, f)


# -- C5: 512 independent 512^2 grids, K=1000 each, tau 0.5 --------------------

def c5(seed: int = 0, items: int = 512, n: int = 512, k: int = 1000, first: int = 0):
    grid = GridSpec((0.0, 0.0), 1.0, (n, n))
    pss = [random_node_sources(seed + i, grid, k) for i in range(first, first + items)]
    return {"grid": grid, "tau": 0.5, "items": pss}
