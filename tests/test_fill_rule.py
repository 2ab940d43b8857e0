"""The sparse flagged-fill rule (tests/fill_rule.py, implemented per flagged
node by csrc/fill.cu) reproduces scipy.ndimage.distance_transform_edt's
nearest-unflagged indices exactly, ties included, in 1-3 dimensions."""

import numpy as np
from scipy import ndimage

from fill_rule import fill_indices


def _check(mask):
    _, ref = ndimage.distance_transform_edt(mask, return_indices=True)
    got = fill_indices(mask)
    assert np.array_equal(got, ref), (mask.shape, np.argwhere(np.any(got != ref, axis=0))[:5])


def test_fill_rule_random_masks():
    rng = np.random.default_rng(1)
    for _ in range(300):
        rank = int(rng.integers(1, 4))
        shape = tuple(int(x) for x in rng.integers(2, 13 if rank < 3 else 7, rank))
        mask = rng.random(shape) < rng.uniform(0.05, 0.9)
        if mask.all():
            continue
        _check(mask)


def test_fill_rule_dense_blocks_and_full_lines():
    rng = np.random.default_rng(2)
    for _ in range(60):
        rank = int(rng.integers(2, 4))
        shape = tuple(int(x) for x in rng.integers(5, 16 if rank == 2 else 9, rank))
        mask = np.zeros(shape, dtype=bool)
        for _ in range(int(rng.integers(1, 4))):  # solid boxes: long flagged runs, whole lines
            lo = [int(rng.integers(0, s)) for s in shape]
            hi = [int(min(s, l + rng.integers(1, s + 1))) for l, s in zip(lo, shape)]
            mask[tuple(slice(a, b) for a, b in zip(lo, hi))] = True
        if mask.all():
            continue
        _check(mask)


def test_fill_rule_curves_and_shells():
    yy, xx = np.mgrid[0:40, 0:37]
    for r in (3.0, 7.5, 12.2, 17.0):
        for w in (0.5, 0.75, 1.5):
            _check(np.abs(np.hypot(yy - 19.3, xx - 17.8) - r) < w)
    zz, yy, xx = np.mgrid[0:18, 0:17, 0:16]
    for r in (3.0, 6.4):
        _check(np.abs(np.sqrt((zz - 8.6) ** 2 + (yy - 8.1) ** 2 + (xx - 7.7) ** 2) - r) < 0.9)
