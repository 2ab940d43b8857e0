"""GPU: the slab-decomposed 3-D schedule (ranks emulated in one process, no
cross-rank waiting) reproduces the single-GPU pipeline bit for bit, both with
the NCCL-style exchange (block copies) and with the exchange fused into the
passes (peer-pointer stores into the owners' arenas, EIK_SLAB_P2P)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("world", [1, 2, 4])
def test_emulated_slab_bit_identical(cuda_ok, world, p2p):
    import torch

    from paper_1112_3010_b200 import GridSpec, engine, workloads
    from paper_1112_3010_b200.slab import (CudaSlabExecutor, fill_masks_emulated, local_nodes, run_emulated,
                                           run_emulated_p2p)

    grid = GridSpec((-15.5, -15.5, -15.5), 1.0, (32, 32, 32))
    tau = 0.75
    v, f = workloads.perturbed_sphere(0, freq=12, radius=10.0)
    surf = workloads.surface_from_mesh(v, f)
    rng = np.random.Generator(np.random.PCG64(5))
    nodes = np.sort(rng.choice(grid.num_nodes, 400, replace=False))
    dt = engine.DistanceTransform(grid, tau, grad=True, sign=True)
    sn, sw = dt.sign_inputs(surf)
    ref = dt.run_host(nodes, sign_nodes=sn, sign_weights=sw)

    exs = [CudaSlabExecutor(grid, tau, world, r, p2p=p2p) for r in range(world)]
    lists = []
    for ex in exs:
        ln, _ = local_nodes(nodes, ex.layout)
        lsn, lsw = local_nodes(sn, ex.layout, sw)
        lists.append((ln, lsn, lsw))
    outs = (run_emulated_p2p if p2p else run_emulated)(exs, lists)
    fill_masks_emulated(exs, outs, sn, hd=1)
    torch.cuda.synchronize()
    got = {k: torch.cat([o[k] for o in outs]).cpu().numpy() for k in ("S", "mu", "mask")}
    for a in range(3):
        got[f"g{a}"] = torch.cat([o["grad"][a] for o in outs]).cpu().numpy()
    assert np.array_equal(got["S"], ref["S"], equal_nan=True)
    assert np.array_equal(got["mu"], ref["mu"])
    assert np.array_equal(got["mask"], ref["mask"])
    for a in range(3):
        assert np.array_equal(got[f"g{a}"], ref["grad"][a], equal_nan=True)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_emulated_streamed_slab_matches_eik_run(cuda_ok, world, monkeypatch):
    """The streamed slab schedule (one V pair, one W pair per rank): S and grad S
    bit-identical to eik_run, mu to rounding (it sums its three inputs after the
    inverse transforms), masks equal after the fill; and bit-identical in every
    field to eik_run's own streamed schedule."""
    import torch

    from paper_1112_3010_b200 import GridSpec, engine, workloads
    from paper_1112_3010_b200.slab import CudaSlabExecutor, fill_masks_emulated, local_nodes, run_emulated_streamed

    grid = GridSpec((-15.5, -15.5, -15.5), 1.0, (32, 32, 32))
    tau = 0.75
    v, f = workloads.perturbed_sphere(0, freq=12, radius=10.0)
    surf = workloads.surface_from_mesh(v, f)
    rng = np.random.Generator(np.random.PCG64(5))
    nodes = np.sort(rng.choice(grid.num_nodes, 400, replace=False))
    dt = engine.DistanceTransform(grid, tau, grad=True, sign=True)
    sn, sw = dt.sign_inputs(surf)
    ref = dt.run_host(nodes, sign_nodes=sn, sign_weights=sw)
    monkeypatch.setenv("EIK_STREAM3D", "1")
    ref_s = dt.run_host(nodes, sign_nodes=sn, sign_weights=sw)
    monkeypatch.delenv("EIK_STREAM3D")

    exs = [CudaSlabExecutor(grid, tau, world, r, streamed=True) for r in range(world)]
    lists = []
    for ex in exs:
        ln, _ = local_nodes(nodes, ex.layout)
        lsn, lsw = local_nodes(sn, ex.layout, sw)
        lists.append((ln, lsn, lsw))
    outs = run_emulated_streamed(exs, lists)
    fill_masks_emulated(exs, outs, sn, hd=1)
    torch.cuda.synchronize()
    got = {k: torch.cat([o[k] for o in outs]).cpu().numpy() for k in ("S", "mu", "mask")}
    assert np.array_equal(got["S"], ref["S"], equal_nan=True)
    assert np.abs(got["mu"] - ref["mu"]).max() <= 1e-12
    assert np.array_equal(got["mu"], ref_s["mu"])
    assert np.array_equal(got["mask"], ref["mask"])
    for a in range(3):
        ga = torch.cat([o["grad"][a] for o in outs]).cpu().numpy()
        assert np.array_equal(ga, ref["grad"][a], equal_nan=True)


def test_p2p_slab_repeat_and_validation(cuda_ok):
    """Two consecutive steps through the same arenas agree; geometry is checked."""
    import torch

    from paper_1112_3010_b200 import GridSpec, ValidationError
    from paper_1112_3010_b200._native import NativeError
    from paper_1112_3010_b200.slab import CudaSlabExecutor, local_nodes, run_emulated_p2p

    grid = GridSpec((0.0, 0.0, 0.0), 1.0, (16, 12, 10))
    rng = np.random.Generator(np.random.PCG64(9))
    nodes = np.sort(rng.choice(grid.num_nodes, 60, replace=False))
    exs = [CudaSlabExecutor(grid, 1.0, 2, r, sign=False, p2p=True) for r in range(2)]
    lists = [(local_nodes(nodes, ex.layout)[0], None, None) for ex in exs]
    a = run_emulated_p2p(exs, lists)
    b = run_emulated_p2p(exs, lists)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x["S"], y["S"])
    with pytest.raises((ValidationError, NativeError)):
        exs[0].plan.slab_finish(None, 3, exs[0].layout.ks, S=a[0]["S"], p2p=True)


@pytest.mark.parametrize("mode", ["nccl", "p2p", "streamed"])
@pytest.mark.parametrize("world", [2, 4])
def test_emulated_slab_long_axis0_bit_identical(cuda_ok, world, mode):
    """Axis 0 padded to 1024 points: the ranks' axis-0 column kernels read their k1 slab of the
    LINE-MAJOR kernel spectra (KSpec::ls) in the wide 3-D configuration, and the lines kernels
    run 16 values per thread; every schedule must still reproduce eik_run bit for bit."""
    import torch

    from paper_1112_3010_b200 import GridSpec, engine
    from paper_1112_3010_b200.slab import (CudaSlabExecutor, fill_masks_emulated, local_nodes, run_emulated,
                                           run_emulated_p2p, run_emulated_streamed)

    grid = GridSpec((0.0, 0.0, 0.0), 1.0, (512, 16, 12))  # the peer-store schedule wants c0 / G a power of two
    tau = 12.0
    rng = np.random.Generator(np.random.PCG64(11))
    N = grid.num_nodes
    nodes = np.sort(rng.choice(N, 900, replace=False))
    sn = np.sort(rng.choice(N, 700, replace=False))
    sw = rng.standard_normal((3, sn.size))
    dt = engine.DistanceTransform(grid, tau, grad=True, sign=True)
    ref = dt.run_host(nodes, sign_nodes=sn, sign_weights=sw)

    streamed = mode == "streamed"
    exs = [CudaSlabExecutor(grid, tau, world, r, p2p=(mode == "p2p"), streamed=streamed) for r in range(world)]
    lists = []
    for ex in exs:
        ln, _ = local_nodes(nodes, ex.layout)
        lsn, lsw = local_nodes(sn, ex.layout, sw)
        lists.append((ln, lsn, lsw))
    run = run_emulated_streamed if streamed else (run_emulated_p2p if mode == "p2p" else run_emulated)
    outs = run(exs, lists)
    fill_masks_emulated(exs, outs, sn, hd=1)
    torch.cuda.synchronize()
    got = {k: torch.cat([o[k] for o in outs]).cpu().numpy() for k in ("S", "mu", "mask")}
    assert np.array_equal(got["S"], ref["S"], equal_nan=True)
    if streamed:
        assert np.abs(got["mu"] - ref["mu"]).max() <= 1e-12 * max(1.0, np.abs(ref["mu"]).max())
    else:
        assert np.array_equal(got["mu"], ref["mu"])
    assert np.array_equal(got["mask"], ref["mask"])
    for a in range(3):
        ga = torch.cat([o["grad"][a] for o in outs]).cpu().numpy()
        assert np.array_equal(ga, ref["grad"][a], equal_nan=True)
