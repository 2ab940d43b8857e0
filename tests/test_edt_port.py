"""The EDT feature-transform restatement (the algorithm the GPU classify fill
implements) reproduces scipy.ndimage.distance_transform_edt indices exactly,
ties included, in 1-3 dimensions."""

import numpy as np
from scipy import ndimage

from edt_port import edt_indices


def test_edt_port_matches_scipy_random_masks():
    rng = np.random.default_rng(0)
    for _ in range(120):
        rank = int(rng.integers(1, 4))
        shape = tuple(int(x) for x in rng.integers(2, 9 if rank < 3 else 6, rank))
        mask = rng.random(shape) < rng.uniform(0.05, 0.85)
        if mask.all():
            continue
        _, ref = ndimage.distance_transform_edt(mask, return_indices=True)
        assert np.array_equal(edt_indices(mask), ref), (shape, mask.astype(int))


def test_edt_port_thin_curve_ties():
    # a flagged ring: every flagged node has several equidistant unflagged neighbours
    yy, xx = np.mgrid[0:24, 0:24]
    mask = np.abs(np.hypot(yy - 11.5, xx - 11.5) - 7.0) < 0.75
    _, ref = ndimage.distance_transform_edt(mask, return_indices=True)
    assert np.array_equal(edt_indices(mask), ref)
