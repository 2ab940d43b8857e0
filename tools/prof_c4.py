"""ncu driver: C4 at --size^3 (default 1024) through eik_run, W warm-up + K steps, device-resident."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

from paper_1112_3010_b200 import _native
from paper_1112_3010_b200 import workloads as wl
from paper_1112_3010_b200.engine import field_bits

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d = wl.c4(0, n=n)
grid = d["grid"]
N = grid.num_nodes
dev = torch.device("cuda", 0)
plan = _native.Plan(3, grid.counts, grid.spacing, d["tau"], field_bits(3, True, False, True), 0)
nd, sn, sw = (torch.as_tensor(np.ascontiguousarray(d[k]), device=dev) for k in ("nodes", "sign_nodes", "sign_weights"))
S, mu = (torch.empty(N, dtype=torch.float64, device=dev) for _ in range(2))
mask = torch.empty(N, dtype=torch.uint8, device=dev)
grad = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(3)]
for _ in range(steps):
    plan.run(nd, None, 1, sn, sw, S=S, grad=grad, mu=mu, mask=mask, host=False)
torch.cuda.synchronize()
print("ok", n, plan.info())
