"""Persistent launches (one resident wave of CTAs walking the tile list, the row
feed running across tiles) against one CTA per tile: bit-identical fields.
EIK_PERSIST is read once per process, so each setting runs in its own process."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1112_3010_b200 import GridSpec, engine, workloads
out = {}
# 2-D, 1024-point lines (col_tmem<10>, row_kernel<9>), Hessian + winding sign, odd sizes
d = workloads.c2(seed=3, n=300, k=2200, radius=90.0, tau=1.5)
dt = engine.DistanceTransform(d["grid"], d["tau"], grad=True, hess=True, sign=True)
sn, sw = dt.sign_inputs(d["curve"])
r = dt.run_host(d["points"].distinct_nodes(), sign_nodes=sn, sign_weights=sw)
for k in ("S", "mu", "mask"):
    out["a_" + k] = r[k]
for i, g in enumerate(r["grad"] + r["hess"]):
    out[f"a_f{i}"] = g
# 2-D batch of 5 items, 512-point lines
grid = GridSpec((0.0, 0.0), 1.0, (200, 140))
rng = np.random.default_rng(8)
nodes = [np.sort(rng.choice(grid.num_nodes, 300, replace=False)) for _ in range(5)]
offs = np.cumsum([0] + [len(n) for n in nodes])
r = engine.DistanceTransform(grid, 1.0, grad=True).run_host(np.concatenate(nodes), item_offsets=offs)
out["b_S"] = r["S"]
out["b_g0"], out["b_g1"] = r["grad"]
# 3-D with a 512-point axis 0 (col_tmem<9> along axis 0), degree sign
grid = GridSpec((0.0, 0.0, 0.0), 1.0, (140, 12, 10))
nodes = np.sort(rng.choice(grid.num_nodes, 500, replace=False))
w = rng.standard_normal((3, nodes.size))
r = engine.DistanceTransform(grid, 1.25, grad=True, sign=True).run_host(nodes, sign_nodes=nodes, sign_weights=w)
out["c_S"], out["c_mu"], out["c_mask"] = r["S"], r["mu"], r["mask"]
for i, g in enumerate(r["grad"]):
    out[f"c_g{i}"] = g
np.savez(sys.argv[2], **out)
"""


def test_persistent_and_per_tile_launches_bit_identical(cuda_ok, tmp_path):
    res = {}
    for mode in ("0", "1"):
        env = dict(os.environ, EIK_PERSIST=mode)
        path = os.path.join(str(tmp_path), f"p{mode}.npz")
        p = subprocess.run([sys.executable, "-c", SCRIPT, REPO, path], env=env, capture_output=True, text=True,
                           timeout=900)
        assert p.returncode == 0, p.stderr[-3000:]
        res[mode] = np.load(path)
    assert set(res["0"].files) == set(res["1"].files) and len(res["0"].files) == 17
    for k in res["0"].files:
        assert np.array_equal(res["0"][k], res["1"][k], equal_nan=True), k
