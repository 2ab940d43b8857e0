"""Experiment-protocol helpers of R/experiments.py (seeded trials, protocol
grids, node-source draws) for the drivers built on the GPU pipeline.

RNG discipline as the reference (R/experiments.py:1-8, 47-59): trial t of an
experiment seeded with s uses PCG64(s + t).
"""

from __future__ import annotations

import numpy as np

from .grid import GridSpec, PointSet

TAU_SWEEP_VALUES = tuple(5e-5 * (i + 1) for i in range(9))  # R/experiments.py:44


def trial_rng(seed: int, trial: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed + trial))


def _grid_2d(n: int, origin: float, spacing: float) -> GridSpec:
    return GridSpec(origin=(origin, origin), spacing=spacing, counts=(n, n))


def draw_node_sources(rng: np.random.Generator, grid: GridSpec, draws: int) -> PointSet:
    """Node indices drawn with replacement, duplicates collapsed (R/experiments.py:55-59)."""
    idx = np.unique(rng.integers(0, grid.num_nodes, size=draws))
    return PointSet.from_node_indices(grid, idx)
