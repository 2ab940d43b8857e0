"""Example-1 protocol (R/experiments.py:74-168) on the GPU tau sweep against the
same protocol evaluated with the oracle's convolution, trial by trial."""

import math

import numpy as np
import pytest

import eikfld_oracle as orc

pytestmark = pytest.mark.gpu


def test_example1_rows_match_oracle_protocol(cuda_ok):
    from paper_1112_3010_b200 import PrecisionError, experiments
    from paper_1112_3010_b200.distance import r_exact

    taus = (1.0e-3, 1.5e-3, 2.0e-3)  # float64-feasible on the 125 x 125, h = 1/512 protocol grid
    rep = experiments.tau_sweep(trials=2, seed=3, taus=taus)
    assert rep.name == "example1" and len(rep.rows) == 3
    grid = experiments._grid_2d(125, -0.121, 1.0 / 512.0)
    means = np.zeros((2, 3))
    for t in range(2):
        ps = experiments.draw_node_sources(experiments.trial_rng(3, t), grid, 5000)
        exact = r_exact(ps.points, grid).values
        for i, tau in enumerate(taus):
            ref = orc.run_config_unchecked(ps.distinct_nodes(), grid.counts, grid.spacing, tau)
            inc = exact > 0
            means[t, i] = (100.0 * np.abs(ref["S"] - exact)[inc] / exact[inc]).sum() / exact.size
    for i, row in enumerate(rep.rows):
        assert row["tau"] == taus[i]
        assert math.isclose(row["mean_error_pct"], means[:, i].mean(), rel_tol=1e-7)
        assert row["bound_holds"]
    assert rep.rows[1]["sublinear_vs_tau"] in (True, False)
    # the published tau values are below the float64 floor: same error as the reference's native path
    with pytest.raises(PrecisionError):
        experiments.tau_sweep(trials=1, seed=0)
