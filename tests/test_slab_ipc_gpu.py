"""GPU: the fused peer-to-peer slab schedule across PROCESSES (world 2, both on
cuda:0): arenas shared through CUDA IPC handles exchanged over gloo, the
passes storing into the peer's arena, host-side barriers (no kernel ever waits
on another rank).  Checked bit for bit against the single-GPU pipeline."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

COUNTS = (32, 32, 32)
TAU = 0.75


def _inputs():
    from paper_1112_3010_b200 import GridSpec, engine, workloads

    grid = GridSpec((-15.5, -15.5, -15.5), 1.0, COUNTS)
    v, f = workloads.perturbed_sphere(0, freq=12, radius=10.0)
    surf = workloads.surface_from_mesh(v, f)
    rng = np.random.Generator(np.random.PCG64(5))
    nodes = np.sort(rng.choice(grid.num_nodes, 400, replace=False))
    dt = engine.DistanceTransform(grid, TAU, grad=True, sign=True)
    sn, sw = dt.sign_inputs(surf)
    return grid, dt, nodes, sn, sw


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    from paper_1112_3010_b200.slab import CudaSlabExecutor, connect_p2p, fill_rank, local_nodes, run_rank_p2p

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid, _, nodes, sn, sw = _inputs()
    ex = CudaSlabExecutor(grid, TAU, world, rank, p2p=True, device=0)
    connect_p2p(ex, dist)  # IPC handles over gloo; opens the peer's arena

    def barrier():  # host-side: the rank's queued passes are complete before the peer proceeds
        torch.cuda.synchronize()
        dist.barrier()

    ln, _ = local_nodes(nodes, ex.layout)
    lsn, lsw = local_nodes(sn, ex.layout, sw)
    for _ in range(2):  # two steps through the same arenas
        out = run_rank_p2p(ex, barrier, ln, lsn, lsw)
    torch.cuda.synchronize()
    fill_rank(ex, out, sn, dist, hd=1)  # mask halos over gloo (host copies); hd=1 exercises the widening
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), S=out["S"].cpu().numpy(), mu=out["mu"].cpu().numpy(),
             mask=out["mask"].cpu().numpy(), **{f"g{a}": out["grad"][a].cpu().numpy() for a in range(3)})
    barrier()  # the peer is done storing into / reading from this rank's arena
    dist.destroy_process_group()


def test_p2p_slab_two_processes_ipc(cuda_ok):
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        got = {k: np.concatenate([p[k] for p in parts]) for k in ("S", "mu", "mask", "g0", "g1", "g2")}
    _, dt, nodes, sn, sw = _inputs()
    ref = dt.run_host(nodes, sign_nodes=sn, sign_weights=sw)
    assert np.array_equal(got["S"], ref["S"], equal_nan=True)
    assert np.array_equal(got["mu"], ref["mu"])
    assert np.array_equal(got["mask"], ref["mask"])
    for a in range(3):
        assert np.array_equal(got[f"g{a}"], ref["grad"][a], equal_nan=True)
