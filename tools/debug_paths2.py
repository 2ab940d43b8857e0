import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import eikfld_oracle as orc
from paper_1112_3010_b200 import engine, workloads
d = workloads.c2(seed=2, n=512, k=4096, radius=150.0, tau=2.0)
grid = d["grid"]
nodes = d["points"].distinct_nodes()
ref = orc.run_config_unchecked(nodes, grid.counts, 1.0, 2.0, want_hessian=True)
keep = ref["phi"] >= 1e-5 * ref["phi"].max()
for hess in (False, True):
    for sign in (False, True):
        dt = engine.DistanceTransform(grid, 2.0, grad=True, hess=hess, sign=sign)
        kw = {}
        if sign:
            sn, sw = dt.sign_inputs(d["curve"]); kw = dict(sign_nodes=sn, sign_weights=sw)
        out = dt.run_host(nodes, **kw)
        err = (np.abs(out["S"] - ref["S"])[keep] / np.maximum(np.abs(ref["S"][keep]), 1)).max()
        print("hess", hess, "sign", sign, os.environ.get("EIK_TMEM"), "S err", err)
