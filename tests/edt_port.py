"""Pure-Python restatement of scipy.ndimage's Euclidean feature transform
(ni_morphology.c _ComputeFT/_VoronoiFT, sampling=None) — TEST INFRASTRUCTURE.

It documents the exact algorithm (and tie rules) the GPU flagged-fill in
paper_1112_3010_b200/csrc/classify.cu implements; test_edt_port.py checks it
against scipy itself on random masks.
"""
import numpy as np

def voronoi_ft(f_line, coor, d, rank):
    """f_line: list of feature coords (or None) along a line; returns new list. Port of scipy _VoronoiFT (sampling=None)."""
    L = len(f_line)
    g = []
    for ii in range(L):
        if f_line[ii] is not None:
            fi = f_line[ii]
            fd = fi[d]
            wR = 0.0
            for jj in range(rank):
                if jj != d:
                    tw = fi[jj] - coor[jj]
                    wR += tw * tw
            while len(g) >= 2:
                idx1 = g[-1]; idx2 = g[-2]
                f1 = f_line[idx1][d]
                a = f1 - f_line[idx2][d]
                b = fd - f1
                c = a + b
                uR = vR = 0.0
                for jj in range(rank):
                    if jj != d:
                        tu = f_line[idx2][jj] - coor[jj]
                        tv = f_line[idx1][jj] - coor[jj]
                        uR += tu * tu; vR += tv * tv
                if c * vR - b * uR - a * wR - a * b * c <= 0.0:
                    break
                g.pop()
            g.append(ii)
    out = [None] * L
    if g:
        l = 0; maxl = len(g) - 1
        for ii in range(L):
            def dist(idx):
                s = 0.0
                for jj in range(rank):
                    t = (f_line[idx][jj] - ii) if jj == d else (f_line[idx][jj] - coor[jj])
                    s += t * t
                return s
            delta1 = dist(g[l])
            while l < maxl:
                delta2 = dist(g[l + 1])
                if delta1 <= delta2:
                    break
                delta1 = delta2
                l += 1
            out[ii] = f_line[g[l]]
    return out

def edt_indices_2d(mask):
    n0, n1 = mask.shape
    F = [[None] * n1 for _ in range(n0)]
    # d = 0: for each column (fixed coor[1]) along axis 0
    for j in range(n1):
        line = [None if mask[i, j] else (i, j) for i in range(n0)]
        res = voronoi_ft(line, (0, j), 0, 2)
        for i in range(n0):
            F[i][j] = res[i]
    # d = 1: for each row (fixed coor[0]) along axis 1
    for i in range(n0):
        line = [F[i][j] for j in range(n1)]
        res = voronoi_ft(line, (i, 0), 1, 2)
        for j in range(n1):
            F[i][j] = res[j]
    idx = np.zeros((2, n0, n1), dtype=np.int64)
    for i in range(n0):
        for j in range(n1):
            idx[0, i, j], idx[1, i, j] = F[i][j]
    return idx



def edt_indices(mask):
    """Nearest background (False) index per element, any rank 1-3."""
    mask = np.asarray(mask, dtype=bool)
    rank = mask.ndim
    shape = mask.shape
    F = np.full(shape + (rank,), -1, dtype=np.int64)
    for idx in np.ndindex(*shape):
        if not mask[idx]:
            F[idx] = idx
    for d in range(rank):
        other = [range(n) for a, n in enumerate(shape) if a != d]
        for rest in np.ndindex(*[n for a, n in enumerate(shape) if a != d]):
            coor = list(rest)
            coor.insert(d, 0)
            sl = list(coor)
            line = []
            for ii in range(shape[d]):
                sl[d] = ii
                f = F[tuple(sl)]
                line.append(None if f[0] < 0 else tuple(int(x) for x in f))
            res = voronoi_ft(line, coor, d, rank)
            for ii in range(shape[d]):
                sl[d] = ii
                if res[ii] is not None:
                    F[tuple(sl)] = res[ii]
    return np.moveaxis(F, -1, 0)
