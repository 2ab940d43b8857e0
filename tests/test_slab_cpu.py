"""Slab-decomposed 3-D schedule over world_size 2 on CPU (gloo all-to-all),
numpy executor, against the oracle.  Covers node partitioning, the packed
[dest][plane][k1'][k2] layouts, the two exchanges and the reassembly."""

import math
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import eikfld_oracle as orc
from conftest import rng_for

COUNTS = (8, 6, 5)
H_SP = 0.5
TAU = 1.5


def _inputs():
    rng = rng_for(11)
    N = int(np.prod(COUNTS))
    nodes = np.sort(rng.choice(N, 20, replace=False))
    snodes = np.sort(rng.choice(N, 15, replace=False))
    sw = rng.standard_normal((3, snodes.size))
    return nodes, snodes, sw


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, p2p=False):
    import torch
    import torch.distributed as dist

    from paper_1112_3010_b200.slab import local_nodes, run_rank, run_rank_p2p, run_rank_streamed
    from slab_numpy import NumpyP2PSlabExecutor, NumpySlabExecutor, NumpyStreamedSlabExecutor

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    streamed = p2p == "streamed"
    p2p = p2p is True
    cls = NumpyStreamedSlabExecutor if streamed else (NumpyP2PSlabExecutor if p2p else NumpySlabExecutor)
    ex = cls(COUNTS, H_SP, TAU, world, rank)
    nodes, snodes, sw = _inputs()
    ln, _ = local_nodes(nodes, ex.layout)
    lsn, lsw = local_nodes(snodes, ex.layout, sw)
    if p2p:
        names = [None] * world
        dist.all_gather_object(names, ex.name)
        ex.connect(names)
        dist.barrier()
        out = run_rank_p2p(ex, dist.barrier, ln, lsn, lsw)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), S=out["S"], phi=out["phi"], mu=out["mu"],
                 gx=out["grad"][0], gy=out["grad"][1], gz=out["grad"][2])
        dist.barrier()  # every peer is done with this rank's arena
        ex.close()
        dist.destroy_process_group()
        return

    def exchange(send, recv):
        for s, r in zip(send, recv):
            rt = torch.from_numpy(r.view(np.float64))
            dist.all_to_all_single(rt, torch.from_numpy(np.ascontiguousarray(s).view(np.float64)))

    out = (run_rank_streamed if streamed else run_rank)(ex, exchange, ln, lsn, lsw)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), S=out["S"], phi=out["phi"], mu=out["mu"],
             gx=out["grad"][0], gy=out["grad"][1], gz=out["grad"][2])
    dist.destroy_process_group()


@pytest.mark.parametrize("p2p", [False, True, "streamed"])
@pytest.mark.parametrize("world", [2])
def test_slab_schedule_world2_gloo(world, p2p):
    """NCCL-style all-to-all schedule, the fused peer-store schedule and the
    streamed (one input / one component at a time) schedule."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, p2p), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        got = {k: np.concatenate([p[k] for p in parts]) for k in ("S", "phi", "mu", "gx", "gy", "gz")}
    nodes, snodes, sw = _inputs()
    ref = orc.run_config_unchecked(nodes, COUNTS, H_SP, TAU)
    scale = np.abs(ref["phi"]).max()
    assert np.abs(got["phi"] - ref["phi"]).max() <= 1e-12 * scale
    for a, k in enumerate(("gx", "gy", "gz")):
        assert np.abs(got[k] - ref["grad"][a]).max() <= 1e-9
    # degree-type sum with the same weighted impulses, oracle engine
    ks = [orc.ratio_kernel(COUNTS, H_SP, a, 3) for a in range(3)]
    conv = orc.Convolver(COUNTS, ks[0].shape)
    mu_ref = 0.0
    for a in range(3):
        g = np.zeros(int(np.prod(COUNTS)))
        g[snodes] = sw[a]
        mu_ref = mu_ref + conv.convolve(ks[a], g.reshape(COUNTS)).reshape(-1)
    mu_ref = -mu_ref / (4.0 * math.pi)
    assert np.abs(got["mu"] - mu_ref).max() <= 1e-12 * max(1.0, np.abs(mu_ref).max())


def test_layout_partition():
    from paper_1112_3010_b200.slab import SlabLayout, local_nodes

    L = SlabLayout(COUNTS, (16, 16, 16), 2, 1)
    assert (L.c0loc, L.ks, L.H, L.i0_begin, L.k1_begin) == (4, 8, 9, 4, 8)
    nodes = np.array([0, 29, 30, 119, 120, 239])
    ln, _ = local_nodes(nodes, L)
    assert list(ln) == [0, 119]  # 120 and 239 re-based by 4 planes * 30 nodes
    with pytest.raises(Exception):
        SlabLayout((7, 6, 5), (16, 16, 16), 2, 0)
