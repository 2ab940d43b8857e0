"""Locate wrong outputs of the 3-D engine path with index-coded kernels (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import eikfld_oracle as orc
from paper_1112_3010_b200 import _native

for counts in [(9, 10), (9, 3), (17, 5), (5, 17), (6, 9, 7), (6, 16, 7), (4, 9, 4), (9, 4, 4), (4, 4, 9), (4, 17, 4), (4, 5, 4), (12, 12, 12)]:
    ks = tuple(2 * c - 1 for c in counts)
    rng = np.random.Generator(np.random.PCG64(1))
    kern = rng.random(ks)
    for field_kind in ("delta",):
        field = np.zeros(counts)
        if field_kind == "delta":
            field[(0,) * len(counts)] = 1.0
        else:
            field = rng.random(counts)
        got = _native.convolve(counts, kern[None], field)[0].reshape(counts)
        ref = orc.Convolver(counts, ks).convolve(kern, field)
        err = np.abs(got - ref)
        bad = np.argwhere(err > 1e-12 * np.abs(ref).max())
        print(counts, field_kind, "max err", err.max(), "bad", len(bad), "first", bad[:6].tolist())
