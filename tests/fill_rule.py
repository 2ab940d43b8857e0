"""Sparse restatement of scipy's EDT feature transform for flagged-node fill
(test infrastructure; the rule csrc/fill.cu implements per flagged node).

scipy.ndimage.distance_transform_edt(flagged, return_indices=True) runs one
Voronoi lower-envelope pass per axis (ni_morphology.c _VoronoiFT, axis 0
first).  With integer coordinates every comparison in that pass is exact, and
its result at a node p of the line along axis d is:

  * p unflagged: p itself (its own feature is at distance 0);
  * p flagged:   F_{d-1}(q*) where q* is the line member of SMALLEST position
                 among those whose pass-(d-1) feature minimises the full
                 squared distance to p (line members without a feature are
                 skipped; pass -1 features are the unflagged nodes themselves).

(Minimisers at p are never popped from the envelope stack, and the query walk
stops at the first of them.)  Only members with (offset)^2 <= best distance
can tie or win, so the scan stops there: the rule touches O(local) nodes per
flagged node instead of whole lines.
"""

import numpy as np


def _feat(flag, coord, d):
    """Feature (tuple of coordinates) of `coord` after the pass along axis d, or None."""
    if not flag[coord]:
        return coord
    if d < 0:
        return None
    n = flag.shape[d]
    x0 = coord[d]
    best = None  # (dist, position, feature)
    t = 0
    while True:
        if best is not None and t * t > best[0]:
            break
        if x0 - t < 0 and x0 + t >= n:
            break
        for x in ((x0 - t, x0 + t) if t else (x0,)):
            if not 0 <= x < n:
                continue
            q = coord[:d] + (x,) + coord[d + 1:]
            f = _feat(flag, q, d - 1)
            if f is None:
                continue
            dist = sum((fa - ca) ** 2 for fa, ca in zip(f, coord))
            if best is None or (dist, x) < (best[0], best[1]):
                best = (dist, x, f)
        t += 1
    return None if best is None else best[2]


def fill_indices(flag):
    """Index array shaped like scipy's `return_indices` output (rank, *shape)."""
    flag = np.asarray(flag, dtype=bool)
    rank = flag.ndim
    out = np.indices(flag.shape)
    for coord in zip(*np.nonzero(flag)):
        coord = tuple(int(c) for c in coord)
        f = _feat(flag, coord, rank - 1)
        if f is None:
            continue
        for a in range(rank):
            out[(a,) + coord] = f[a]
    return out
