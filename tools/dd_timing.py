"""Time the double-double path (host in / host out, synchronous) on C1-like
and larger 2-D grids: python tools/dd_timing.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1112_3010_b200 import GridSpec, _native

for n, k in ((256, 2000), (512, 2000), (1024, 4000)):
    grid = GridSpec((0.0, 0.0), 1.0, (n, n))
    nodes = np.sort(np.random.Generator(np.random.PCG64(0)).choice(n * n, k, replace=False))
    for fields, label in ((_native.FIELD_PHI | _native.FIELD_S, "S"),
                          (_native.FIELD_PHI | _native.FIELD_S | _native.FIELD_GRAD, "S+grad")):
        t0 = time.perf_counter()
        plan = _native.DDPlan(2, (n, n), 1.0, 0.5, fields)
        tp = time.perf_counter() - t0
        S = np.empty(n * n)
        g = [np.empty(n * n), np.empty(n * n)] if "grad" in label else (None, None, None)
        plan.run(nodes, S=S, grad=g)
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            plan.run(nodes, S=S, grad=g)
        dt = (time.perf_counter() - t0) / reps
        print(f"DD {n}^2 {label}: plan {tp:.2f} s, run {dt * 1e3:.1f} ms, {n * n / dt / 1e6:.1f} Mpts/s")
        plan.close()
