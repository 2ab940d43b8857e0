import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import eikfld_oracle as orc
from paper_1112_3010_b200 import engine, GridSpec
for counts in [(512, 64), (256, 64), (1024, 32), (64, 512), (600, 40), (300, 40)]:
    grid = GridSpec((0.0, 0.0), 1.0, counts)
    nodes = np.sort(np.random.default_rng(1).choice(grid.num_nodes, 200, replace=False))
    dt = engine.DistanceTransform(grid, 2.0, grad=True)
    out = dt.run_host(nodes)
    ref = orc.run_config_unchecked(nodes, counts, 1.0, 2.0)
    keep = ref["phi"] >= 1e-5 * ref["phi"].max()
    err = (np.abs(out["S"] - ref["S"])[keep] / np.maximum(np.abs(ref["S"][keep]), 1)).max()
    print(counts, os.environ.get("EIK_TMEM"), os.environ.get("EIK_ROWDFT"), "S rel err", err)
