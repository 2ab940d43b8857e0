"""Short driver for ncu: plan + W warm-up + K steps of one config, device-resident (no timing)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

import bench
from paper_1112_3010_b200 import _native
from paper_1112_3010_b200.engine import field_bits

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = bench.build_workload(cfg, 0, 0, 1, 512)
grid = w["grid"]
dim = len(grid.counts)
plan = _native.Plan(dim, grid.counts, grid.spacing, w["tau"],
                    field_bits(dim, w.get("grad", False), w.get("hess", False), w.get("sign") is not None), 0)
dev = torch.device("cuda", 0)
B = len(w["nodes"])
N = grid.num_nodes
nodes = torch.from_numpy(np.concatenate(w["nodes"])).to(dev)
offs = torch.from_numpy(np.cumsum([0] + [len(n) for n in w["nodes"]]).astype(np.int64)).to(dev) if B > 1 else None
sn = sw = None
if w.get("sign") is not None:
    sn = torch.from_numpy(w["sign"][0]).to(dev)
    sw = torch.from_numpy(w["sign"][1]).to(dev)
f64 = lambda: torch.empty(B * N, dtype=torch.float64, device=dev)  # noqa: E731
S = f64()
grad = [f64() for _ in range(dim)]
hess = [f64() for _ in range(3)] if w.get("hess") else (None,) * 3
mu = f64() if sn is not None else None
mask = torch.empty(B * N, dtype=torch.uint8, device=dev) if sn is not None else None
for _ in range(steps):
    plan.run(nodes, offs, B, sn, sw, S=S, grad=grad, hess=hess, mu=mu, mask=mask, host=False)
torch.cuda.synchronize()
print("ok", cfg, plan.info())
