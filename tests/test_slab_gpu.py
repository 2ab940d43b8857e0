"""GPU: the slab-decomposed 3-D schedule (ranks emulated in one process, no
cross-rank waiting) reproduces the single-GPU pipeline bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 4])
def test_emulated_slab_bit_identical(cuda_ok, world):
    import torch

    from paper_1112_3010_b200 import GridSpec, engine, workloads
    from paper_1112_3010_b200.slab import CudaSlabExecutor, local_nodes, run_emulated

    grid = GridSpec((-15.5, -15.5, -15.5), 1.0, (32, 32, 32))
    tau = 0.75
    v, f = workloads.perturbed_sphere(0, freq=12, radius=10.0)
    surf = workloads.surface_from_mesh(v, f)
    rng = np.random.Generator(np.random.PCG64(5))
    nodes = np.sort(rng.choice(grid.num_nodes, 400, replace=False))
    dt = engine.DistanceTransform(grid, tau, grad=True, sign=True)
    sn, sw = dt.sign_inputs(surf)
    ref = dt.run_host(nodes, sign_nodes=sn, sign_weights=sw)

    exs = [CudaSlabExecutor(grid, tau, world, r) for r in range(world)]
    lists = []
    for ex in exs:
        ln, _ = local_nodes(nodes, ex.layout)
        lsn, lsw = local_nodes(sn, ex.layout, sw)
        lists.append((ln, lsn, lsw))
    outs = run_emulated(exs, lists)
    torch.cuda.synchronize()
    got = {k: torch.cat([o[k] for o in outs]).cpu().numpy() for k in ("S", "mu", "mask")}
    for a in range(3):
        got[f"g{a}"] = torch.cat([o["grad"][a] for o in outs]).cpu().numpy()
    assert np.array_equal(got["S"], ref["S"], equal_nan=True)
    assert np.array_equal(got["mu"], ref["mu"])
    assert np.array_equal(got["mask"], ref["mask"])
    for a in range(3):
        assert np.array_equal(got[f"g{a}"], ref["grad"][a], equal_nan=True)
