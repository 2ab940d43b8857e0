"""Small-grid workload for compute-sanitizer (memcheck / racecheck / synccheck).

Exercises every device code path on grids small enough that the sanitizers
finish in minutes: 2-D S+grad+Hessian+winding (TMEM column kernels, mbarrier
row feed), batches with ragged items, 3-D gradient + degree (lines kernels),
the tau sweep, classify, the double-double path, the emulated slab schedules
(peer stores, G = 2) and CUDA-graph replay.  Usage:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [part ...]
"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402


def part_2d():
    from paper_1112_3010_b200 import engine, workloads

    d = workloads.c2(seed=1, n=96, k=720, radius=28.0, tau=2.0)
    dt = engine.DistanceTransform(d["grid"], 2.0, grad=True, hess=True, sign=True)
    sn, sw = dt.sign_inputs(d["curve"])
    out = dt.run_host(d["points"].distinct_nodes(), sign_nodes=sn, sign_weights=sw)
    assert np.isfinite(out["S"]).all()
    # C2-shaped column kernels (4096-point four-step) at a reduced node count
    d = workloads.c2(seed=0, n=2048, k=2048, radius=600.0, tau=0.5)
    dt = engine.DistanceTransform(d["grid"], 0.5, grad=True, hess=True, sign=True)
    sn, sw = dt.sign_inputs(d["curve"])
    dt.run_host(d["points"].distinct_nodes(), sign_nodes=sn, sign_weights=sw)


def part_batch():
    from paper_1112_3010_b200 import engine
    from paper_1112_3010_b200.grid import GridSpec

    grid = GridSpec((0.0, 0.0), 1.0, (64, 64))
    rng = np.random.default_rng(3)
    items = [np.sort(rng.choice(64 * 64, k, replace=False)) for k in (30, 0, 5, 64)]
    offs = np.cumsum([0] + [len(x) for x in items])
    dt = engine.DistanceTransform(grid, 0.5, grad=True)
    dt.run_host(np.concatenate(items), item_offsets=offs)


def part_3d():
    from paper_1112_3010_b200 import engine, workloads

    d = workloads.c4(seed=0, n=32, radius=10.0, freq=8)
    dt = engine.DistanceTransform(d["grid"], d["tau"], grad=True, sign=True)
    sn, sw = d["sign_nodes"], d["sign_weights"]
    dt.run_host(d["nodes"], sign_nodes=sn, sign_weights=sw)


def part_sweep():
    from paper_1112_3010_b200 import engine, workloads

    d = workloads.c1(seed=0, n=64, k=50)
    engine.TauSweep(d["grid"], [0.5, 1.0, 2.0]).run_host(d["points"].distinct_nodes())


def part_classify():
    from paper_1112_3010_b200 import _native

    rng = np.random.default_rng(0)
    mu = rng.standard_normal(40 * 33)
    fl = np.sort(rng.choice(40 * 33, 100, replace=False))
    _native.classify((40, 33), mu, fl, 1)


def part_dd():
    from paper_1112_3010_b200 import PrecisionConfig, derivatives, workloads

    d = workloads.c1(seed=0, n=32, k=20)
    derivatives.gradient(d["points"], d["grid"], PrecisionConfig.bigfloat(2.0, 106))


def part_slab():
    import torch
    from paper_1112_3010_b200 import workloads
    from paper_1112_3010_b200.slab import CudaSlabExecutor, local_nodes, run_emulated, run_emulated_p2p

    d = workloads.c4(seed=0, n=32, radius=10.0, freq=8)
    for p2p in (False, True):
        exs = [CudaSlabExecutor(d["grid"], d["tau"], 2, r, p2p=p2p) for r in range(2)]
        lists = []
        for ex in exs:
            ln, _ = local_nodes(d["nodes"], ex.layout)
            lsn, lsw = local_nodes(d["sign_nodes"], ex.layout, d["sign_weights"])
            lists.append((ln, lsn, lsw))
        (run_emulated_p2p if p2p else run_emulated)(exs, lists)
    torch.cuda.synchronize()


def part_graph():
    import torch
    from paper_1112_3010_b200 import _native, engine, workloads

    d = workloads.c1(seed=0, n=64, k=50)
    dt = engine.DistanceTransform(d["grid"], 0.5, grad=True)
    nodes = torch.from_numpy(d["points"].distinct_nodes()).cuda()
    S = torch.empty(64 * 64, dtype=torch.float64, device="cuda")
    for _ in range(3):
        dt.plan.run(nodes, S=S, host=False)
    torch.cuda.synchronize()


PARTS = {k[5:]: v for k, v in globals().items() if k.startswith("part_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(PARTS)
    for n in names:
        PARTS[n]()
        print("ok", n, flush=True)
