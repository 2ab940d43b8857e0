"""Slab-decomposed 3-D distance transform across G ranks (BASELINE config C4).

One process per GPU; torch.distributed (NCCL over NVLink/NVSwitch) moves the
data.  Rank r owns:

* real-space planes  i0 in [r*c0/G, (r+1)*c0/G)   (c0 divisible by G), and
* spectral planes    k1 in [r*M1/G, (r+1)*M1/G)   (M1 = padded axis 1).

Per group (distance: delta_Y; sign: the three flux components) the schedule is

  planes  (local)  impulse DFT along axis 2 + FFT along axis 1 of the owned
                   planes -> V packed by destination k1-slab [G][c0/G][ks][H2]
  all-to-all       V  -> [c0][ks][H2] on the owner of the k1-slab
  axis0   (local)  fused axis-0 FFT, kernel-spectrum multiply, inverse per
                   component -> W_j [c0][ks][H2]
and then, for all components together,
  all-to-all       W_j -> [G][c0/G][ks][H2] on the owner of the planes
  finish  (local)  inverse along axis 1, c2r along axis 2, fused epilogue.

So there is one all-to-all per input and one per component, each moving
16 * c0 * M1 * H2 bytes over the whole job.  Every pass is
the same kernel the single-GPU path runs (`eik_run` on a 3-D plan is this
schedule with G = 1), so a G-rank result is bit-identical to the one-GPU
result.  Each rank's plan caches only its k1-slab of the kernel spectra.

The fused variant (`run_rank_p2p`, `CudaSlabExecutor(p2p=True)`) removes the
all-to-alls: the planes and axis-0 kernels store their output blocks straight
into the owning rank's receive arena through CUDA-IPC peer pointers (NVLink /
NVSwitch stores, overlapped with the transforms), leaving two stream-ordered
barriers per step.  It is bit-identical to the NCCL schedule (same kernels,
same arithmetic; only the store addresses differ).

`run_rank` is written against an executor interface (planes / axis0 /
finish plus the V/W buffers) and an `exchange(send, recv)` callable, so the
same orchestration runs with the CUDA executor over NCCL, with several CUDA
executors emulated in one process (`run_emulated`), and with a numpy
executor over gloo in the CPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError


@dataclass(frozen=True)
class SlabLayout:
    counts: tuple
    padded: tuple
    world: int
    rank: int

    def __post_init__(self):
        c0, _, _ = self.counts
        M1 = self.padded[1]
        if c0 % self.world or M1 % self.world:
            raise ValidationError(f"c0={c0} and M1={M1} must be divisible by the {self.world} ranks")

    H = property(lambda self: self.padded[2] // 2 + 1)
    c0loc = property(lambda self: self.counts[0] // self.world)
    ks = property(lambda self: self.padded[1] // self.world)
    i0_begin = property(lambda self: self.rank * self.c0loc)
    k1_begin = property(lambda self: self.rank * self.ks)
    block = property(lambda self: self.c0loc * self.ks * self.H)  # complex elements per peer block
    buf = property(lambda self: self.world * self.block)  # complex elements per V / W buffer
    plane_nodes = property(lambda self: self.counts[1] * self.counts[2])

    def node_range(self):
        lo = self.i0_begin * self.plane_nodes
        return lo, lo + self.c0loc * self.plane_nodes


def local_nodes(nodes, layout: SlabLayout, weights=None):
    """The rank's share of a sorted node list, re-based to its slab; weights (A, K) follow."""
    nodes = np.asarray(nodes, dtype=np.int64)
    lo, hi = layout.node_range()
    a, b = np.searchsorted(nodes, [lo, hi])
    ln = np.ascontiguousarray(nodes[a:b] - lo)
    if weights is None:
        return ln, None
    return ln, np.ascontiguousarray(np.asarray(weights)[:, a:b])


def halo_planes(layout: SlabLayout, hd: int):
    """Planes [e0, e1): the rank's own planes plus up to hd neighbour planes each side."""
    e0 = max(0, layout.i0_begin - hd)
    e1 = min(layout.counts[0], layout.i0_begin + layout.c0loc + hd)
    return e0, e1


def ext_flagged(sign_nodes, layout: SlabLayout, hd: int):
    """Flagged (sign) nodes of planes [e0, e1), flat relative to plane e0."""
    e0, e1 = halo_planes(layout, hd)
    nodes = np.asarray(sign_nodes, dtype=np.int64)
    pl = layout.plane_nodes
    a, b = np.searchsorted(nodes, [e0 * pl, e1 * pl])
    return np.ascontiguousarray(nodes[a:b] - e0 * pl), e0, e1


def fill_masks_emulated(executors, outs, sign_nodes, hd=8):
    """Flagged-node fill of every emulated rank's mask (classify, R/sign.py:179-195):
    each rank reads the neighbours' halo planes straight from their outputs."""
    import torch

    L0 = executors[0].layout
    while True:
        full = torch.cat([o["mask"].view(-1) for o in outs]).view(L0.counts[0], -1)
        try:
            for ex, o in zip(executors, outs):
                ext, e0, e1 = ext_flagged(sign_nodes, ex.layout, hd)
                ex.fill(o, ext, e0, e1, full[e0:e1].contiguous())
            return outs
        except ValidationError:
            if hd >= L0.counts[0]:
                raise
            hd *= 2


def fill_rank(ex, out, sign_nodes, dist, hd=8):
    """Flagged-node fill of one rank's mask: halo planes of the mask from the
    neighbouring ranks (point-to-point), then eik_slab_fill; the halo doubles,
    on every rank at once, until no nearest-unflagged search leaves it."""
    import torch

    L = ex.layout
    G, r = L.world, L.rank
    mask = out["mask"].view(L.c0loc, -1)
    # NCCL moves device tensors; other backends (gloo in the tests) host copies
    wire = mask.device if dist.get_backend() == "nccl" else torch.device("cpu")
    while True:
        h = min(hd, L.c0loc)
        ops = []
        lo = torch.empty((h, mask.shape[1]), dtype=torch.uint8, device=wire) if r > 0 else None
        hi = torch.empty((h, mask.shape[1]), dtype=torch.uint8, device=wire) if r < G - 1 else None
        if r > 0:
            ops += [dist.P2POp(dist.isend, mask[:h].contiguous().to(wire), r - 1), dist.P2POp(dist.irecv, lo, r - 1)]
        if r < G - 1:
            ops += [dist.P2POp(dist.isend, mask[-h:].contiguous().to(wire), r + 1), dist.P2POp(dist.irecv, hi, r + 1)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        parts = [x.to(mask.device) for x in (lo, mask, hi) if x is not None]
        ext, e0, e1 = ext_flagged(sign_nodes, L, h)
        ok = torch.ones(1, device=wire)
        try:
            ex.fill(out, ext, e0, e1, torch.cat(parts).contiguous())
        except ValidationError:
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() > 0:
            return out
        if h >= L.c0loc:
            raise ValidationError("slab fill: a nearest-unflagged search spans more than one neighbour slab")
        hd *= 2


def run_rank(ex, exchange, nodes, sign_nodes=None, sign_weights=None):
    """One rank of the slab schedule.  `nodes` etc. are this rank's local lists."""
    ex.planes(0, nodes, None)
    exchange(ex.V_send[:1], ex.V_recv[:1])
    ex.axis0(0)
    if ex.sign and sign_nodes is not None:
        ex.planes(1, sign_nodes, sign_weights)
        exchange(ex.V_send[:3], ex.V_recv[:3])
        ex.axis0(1)
    exchange(ex.W, ex.W_recv)
    return ex.finish()


def run_rank_streamed(ex, exchange, nodes, sign_nodes=None, sign_weights=None):
    """One rank of the streamed slab schedule (executor built with streamed=True):
    one input and one component at a time through ONE V pair and ONE W pair, so
    C4 at 1024^3 fits two GPUs.  Same all-to-all count as run_rank (one per
    input, one per component); every component returns as a raw real-space field
    and the epilogue runs elementwise at the end."""
    ex.planes_one(0, 0, nodes, None)
    exchange(ex.V_send, ex.V_recv)
    for j in range(ex.n_dist):
        ex.axis0_one(j, accumulate=False)
        exchange(ex.W, ex.W_recv)
        ex.finish_raw(j)
    if ex.sign and sign_nodes is not None:
        for i in range(3):
            ex.planes_one(1, i, sign_nodes, sign_weights)
            exchange(ex.V_send, ex.V_recv)
            ex.axis0_one(4 + i, accumulate=i > 0)
        exchange(ex.W, ex.W_recv)
        ex.finish_raw("mu")
    return ex.epilogue()


def run_emulated_streamed(executors, node_lists):
    """All ranks of the streamed schedule in one process, phase by phase
    (exchanges as block copies); for testing on one device."""
    G = len(executors)

    def swap(send, recv):
        for r in range(G):
            dst = recv(executors[r])[0].view(G, -1)
            for g in range(G):
                dst[g].copy_(send(executors[g])[0].view(G, -1)[r])

    def vswap():
        swap(lambda e: e.V_send, lambda e: e.V_recv)

    def wswap():
        swap(lambda e: e.W, lambda e: e.W_recv)

    for r, ex in enumerate(executors):
        ex.planes_one(0, 0, node_lists[r][0], None)
    vswap()
    for j in range(executors[0].n_dist):
        for ex in executors:
            ex.axis0_one(j, accumulate=False)
        wswap()
        for ex in executors:
            ex.finish_raw(j)
    if executors[0].sign and node_lists[0][1] is not None:
        for i in range(3):
            for r, ex in enumerate(executors):
                ex.planes_one(1, i, node_lists[r][1], node_lists[r][2])
            vswap()
            for ex in executors:
                ex.axis0_one(4 + i, accumulate=i > 0)
        wswap()
        for ex in executors:
            ex.finish_raw("mu")
    return [ex.epilogue() for ex in executors]


def nccl_exchange(dist):
    """exchange(send, recv) = one all_to_all_single per buffer (equal peer blocks)."""

    def exchange(send, recv):
        for s, r in zip(send, recv):
            dist.all_to_all_single(r, s)

    return exchange


def run_rank_p2p(ex, barrier, nodes, sign_nodes=None, sign_weights=None):
    """One rank of the fused peer-to-peer schedule (EIK_SLAB_P2P).

    The planes passes store their k1-slab blocks straight into the owners' V
    slots and the axis-0 passes store their rows straight into the owners' W
    slots (NVLink stores through peer pointers, overlapped with the transforms),
    so the only cross-rank operations are two stream-ordered barriers: after
    the planes passes (every V block landed) and after the axis-0 passes (every
    W block landed).  The distance and sign groups use disjoint slots, so their
    planes passes and their axis-0 passes run back to back.
    """
    ex.planes(0, nodes, None)
    sign = ex.sign and sign_nodes is not None
    if sign:
        ex.planes(1, sign_nodes, sign_weights)
    barrier()
    ex.axis0(0)
    if sign:
        ex.axis0(1)
    barrier()
    return ex.finish()


def stream_barrier(dist, device):
    """Cross-rank barrier ordered on the current stream (one 8-byte all-reduce)."""
    import torch

    flag = torch.zeros(1, dtype=torch.float64, device=device)

    def barrier():
        dist.all_reduce(flag)

    return barrier


def connect_p2p(ex, dist):
    """Exchange the arenas' CUDA IPC handles (one process per GPU) and open the peers."""
    handles = [None] * dist.get_world_size()
    dist.all_gather_object(handles, ex.ipc_handle)
    ex.plan.slab_p2p_connect(ipc_handles=handles)


def run_emulated_p2p(executors, node_lists):
    """All ranks of the peer-to-peer schedule in one process (peer arenas by
    device pointer), phase by phase: no rank ever waits on another."""
    arenas = [ex.arena for ex in executors]
    for ex in executors:
        ex.plan.slab_p2p_connect(peer_arenas=arenas)
    sign = executors[0].sign and node_lists[0][1] is not None
    for r, ex in enumerate(executors):
        ex.planes(0, node_lists[r][0], None)
        if sign:
            ex.planes(1, node_lists[r][1], node_lists[r][2])
    for ex in executors:
        ex.axis0(0)
        if sign:
            ex.axis0(1)
    return [ex.finish() for ex in executors]


def run_emulated(executors, node_lists):
    """All ranks in one process: phase by phase, exchanges as block copies.

    node_lists[r] = (nodes, sign_nodes, sign_weights) local to rank r.  Only
    for testing the decomposition on one device (no rank ever waits on another).
    """
    G = len(executors)

    def swap(get_send, get_recv, n):
        for i in range(n):
            for r in range(G):
                recv = get_recv(executors[r])[i].view(G, -1)
                for g in range(G):
                    recv[g].copy_(get_send(executors[g])[i].view(G, -1)[r])

    for r, ex in enumerate(executors):
        ex.planes(0, node_lists[r][0], None)
    swap(lambda e: e.V_send, lambda e: e.V_recv, 1)
    for ex in executors:
        ex.axis0(0)
    if executors[0].sign and node_lists[0][1] is not None:
        for r, ex in enumerate(executors):
            ex.planes(1, node_lists[r][1], node_lists[r][2])
        swap(lambda e: e.V_send, lambda e: e.V_recv, 3)
        for ex in executors:
            ex.axis0(1)
    swap(lambda e: e.W, lambda e: e.W_recv, len(executors[0].W))
    return [ex.finish() for ex in executors]


class CudaSlabExecutor:
    """CUDA passes of one rank (libeikfld_b200 slab API) with torch device buffers."""

    def __init__(self, grid, tau, world, rank, *, grad=True, sign=True, device=0, p2p=False, streamed=False):
        import torch

        from . import _native
        from .engine import field_bits

        if len(grid.counts) != 3:
            raise ValidationError("the slab decomposition is for 3-D grids")
        probe = _native.Plan(3, grid.counts, grid.spacing, tau, 0, device)
        padded = probe.info()["padded"]
        probe.close()
        self.layout = SlabLayout(tuple(grid.counts), tuple(padded), world, rank)
        L = self.layout
        self.sign = sign
        self.grad = grad
        self.dev = torch.device("cuda", device)
        self.plan = _native.Plan(3, grid.counts, grid.spacing, tau, field_bits(3, grad, False, sign), device,
                                 k1_slab=(L.k1_begin, L.ks))
        n = 2 * L.buf  # doubles per complex buffer
        mk = lambda: torch.empty((L.world, n // L.world), dtype=torch.float64, device=self.dev)  # noqa: E731
        n_in = 3 if sign else 1
        self.n_dist = 1 + (3 if grad else 0)
        n_comp = self.n_dist + (1 if sign else 0)
        self.p2p = p2p
        self.streamed = streamed
        self.N_local = L.c0loc * L.plane_nodes
        if streamed:
            # one V pair and one W pair; the returned component reuses V_send (dead by then)
            if p2p:
                raise ValidationError("the streamed slab schedule uses the all-to-all exchange")
            self.V_send, self.V_recv, self.W = [mk()], [mk()], [mk()]
            self.W_recv = self.V_send
            self._out = None
            return
        if p2p:
            # one arena per rank in the receive layout; the passes store into the
            # owners' arenas, so no send / staging buffers exist at all
            self.arena, self.arena_bytes, self.ipc_handle = self.plan.slab_p2p_init(L.world, L.rank, L.c0loc, L.ks)
            self.V_send = self.V_recv = self.W = self.W_recv = None
            return
        self.V_send = [mk() for _ in range(n_in)]
        self.V_recv = [mk() for _ in range(n_in)]
        self.W = [mk() for _ in range(n_comp)]
        # the spectra V are dead once both axis-0 passes ran: the returned
        # components reuse them (5 + 6 buffers of c0/G * M1 * H2 complex per rank
        # instead of 5 + 5 + 6 -> C4 1024^3 fits 4 or more B200s)
        spare = self.V_send + self.V_recv
        self.W_recv = [spare[j] if j < len(spare) else mk() for j in range(n_comp)]
        self.N_local = L.c0loc * L.plane_nodes

    def _stream(self):
        import torch

        return torch.cuda.current_stream(self.dev).cuda_stream

    def planes(self, group, nodes, weights):
        import torch

        L = self.layout

        def dev(x, dt):
            if x is None or isinstance(x, torch.Tensor):
                return x
            return torch.as_tensor(np.ascontiguousarray(x, dtype=dt), device=self.dev)

        nd = dev(nodes, np.int64)
        wt = dev(weights, np.float64)
        self._keep = (nd, wt)
        if self.p2p:
            self.plan.slab_planes(group, nd, wt, L.c0loc, L.ks, None, self._stream(), p2p=True)
        else:
            self.plan.slab_planes(group, nd, wt, L.c0loc, L.ks, self.V_send[:3 if group else 1], self._stream())

    # -- streamed schedule (run_rank_streamed)
    def _dev(self, x, dt):
        import torch

        if x is None or isinstance(x, torch.Tensor):
            return x
        return torch.as_tensor(np.ascontiguousarray(x, dtype=dt), device=self.dev)

    def _outputs(self):
        import torch

        if self._out is None:
            f = lambda: torch.empty(self.N_local, dtype=torch.float64, device=self.dev)  # noqa: E731
            out = {"S": f(), "underflow": torch.empty(self.N_local, dtype=torch.uint8, device=self.dev)}
            if self.grad:
                out["grad"] = [f() for _ in range(3)]
            if self.sign:
                out["mu"] = f()
                out["mask"] = torch.empty(self.N_local, dtype=torch.uint8, device=self.dev)
            self._out = out
        return self._out

    def planes_one(self, group, inp, nodes, weights):
        L = self.layout
        nd, wt = self._dev(nodes, np.int64), self._dev(weights, np.float64)
        self._keep = (nd, wt)
        self.plan.slab_planes_one(group, inp, nd, wt, L.c0loc, L.ks, self.V_send[0], self._stream())

    def axis0_one(self, kernel, accumulate=False):
        L = self.layout
        self.plan.slab_axis0_one(kernel, self.V_recv[0], L.k1_begin, L.ks, self.W[0], accumulate, self._stream())

    def finish_raw(self, which):
        """Component `which` (0 = phi -> S buffer, 1..3 = gradient numerators, "mu") back to real space, raw."""
        L = self.layout
        out = self._outputs()
        dest = out["mu"] if which == "mu" else (out["S"] if which == 0 else out["grad"][which - 1])
        self.plan.slab_finish_raw(self.W_recv[0], L.c0loc, L.ks, dest, self._stream())

    def epilogue(self):
        out = self._outputs()
        self.plan.slab_epilogue(self.N_local, out["S"], out.get("mu"), S=out["S"], grad=out.get("grad", (None,) * 3),
                                mu=out.get("mu"), mask=out.get("mask"), underflow=out["underflow"],
                                stream=self._stream())
        return out

    def axis0(self, group):
        L = self.layout
        if self.p2p:
            self.plan.slab_axis0(group, None, L.k1_begin, L.ks, None, self._stream(), p2p=True)
            return
        out = [self.W[self.n_dist]] if group else self.W[: self.n_dist]
        self.plan.slab_axis0(group, self.V_recv[:3 if group else 1], L.k1_begin, L.ks, out, self._stream())

    def fill(self, out, ext_nodes, e0, e1, mask_ext):
        """eik_slab_fill: the owned flagged nodes of out["mask"] from the halo-extended mask."""
        import torch

        nd = torch.as_tensor(np.ascontiguousarray(ext_nodes, dtype=np.int64), device=self.dev)
        L = self.layout
        self.plan.slab_fill(nd, e0, e1, L.i0_begin, L.c0loc, mask_ext, out["mask"], self._stream())

    def finish(self):
        import torch

        L = self.layout
        f = lambda: torch.empty(self.N_local, dtype=torch.float64, device=self.dev)  # noqa: E731
        out = {"S": f(), "underflow": torch.empty(self.N_local, dtype=torch.uint8, device=self.dev)}
        if self.grad:
            out["grad"] = [f() for _ in range(3)]
        if self.sign:
            out["mu"] = f()
            out["mask"] = torch.empty(self.N_local, dtype=torch.uint8, device=self.dev)
        self.plan.slab_finish(self.W_recv, L.c0loc, L.ks, S=out["S"], grad=out.get("grad", (None,) * 3),
                              mu=out.get("mu"), mask=out.get("mask"), underflow=out["underflow"],
                              stream=self._stream(), p2p=self.p2p)
        return out
