"""Numpy executor of the slab schedule (TEST INFRASTRUCTURE).

Implements the three slab passes of paper_1112_3010_b200.slab with numpy FFTs
on exactly the buffer layouts the CUDA passes use, so the orchestration
(node partitioning, packing, all-to-all exchanges, reassembly) can be tested
on CPU ranks over gloo.  Kernel samples come from the oracle.
"""

import math

import numpy as np

import eikfld_oracle as orc
from paper_1112_3010_b200.slab import SlabLayout


def _nextpow2(n):
    return 1 << max(1, int(n - 1).bit_length())


def _wrap(centred, counts, padded):
    out = np.zeros(padded)
    idx = [np.r_[0:c, M - (c - 1):M] for c, M in zip(counts, padded)]
    src = [np.r_[c - 1:2 * c - 1, 0:c - 1] for c in counts]
    out[np.ix_(*idx)] = centred[np.ix_(*src)]
    return out


class NumpySlabExecutor:
    def __init__(self, counts, spacing, tau, world, rank, grad=True, sign=True):
        padded = tuple(_nextpow2(2 * c - 1) for c in counts)
        self.layout = L = SlabLayout(tuple(counts), padded, world, rank)
        self.tau, self.grad, self.sign = tau, grad, sign
        base = orc.kernel_exp(counts, spacing, tau)
        fa, _ = orc.directional_kernels(counts, spacing)
        kern = [base] + ([f * base for f in fa] if grad else [])
        sl = slice(L.k1_begin, L.k1_begin + L.ks)
        self.kd = [np.fft.rfftn(_wrap(k, counts, padded))[:, sl, :] for k in kern]
        self.ksg = [np.fft.rfftn(_wrap(orc.ratio_kernel(counts, spacing, a, 3), counts, padded))[:, sl, :]
                    for a in range(3)] if sign else []
        mk = lambda: np.zeros((L.world, L.block), dtype=np.complex128)  # noqa: E731
        n_in = 3 if sign else 1
        self.n_dist = len(kern)
        self.V_send = [mk() for _ in range(n_in)]
        self.V_recv = [mk() for _ in range(n_in)]
        self.W = [mk() for _ in range(self.n_dist + (1 if sign else 0))]
        self.W_recv = [mk() for _ in range(len(self.W))]

    def planes(self, group, nodes, weights):
        L = self.layout
        c0, c1, c2 = L.counts
        M0, M1, M2 = L.padded
        n_in = 3 if group else 1
        for i in range(n_in):
            g = np.zeros(L.c0loc * c1 * c2)
            np.add.at(g, nodes, 1.0 if weights is None else weights[i])
            t = np.fft.fft(np.fft.rfft(g.reshape(L.c0loc, c1, c2), n=M2, axis=2), n=M1, axis=1)
            for dest in range(L.world):
                self.V_send[i][dest] = t[:, dest * L.ks:(dest + 1) * L.ks, :].reshape(-1)

    def axis0(self, group):
        L = self.layout
        c0 = L.counts[0]
        M0 = L.padded[0]
        n_in = 3 if group else 1
        X = [np.fft.fft(self.V_recv[i].reshape(c0, L.ks, L.H), n=M0, axis=0) for i in range(n_in)]
        if group:
            Y = [sum(k * x for k, x in zip(self.ksg, X))]
            dst = [self.W[self.n_dist]]
        else:
            Y = [k * X[0] for k in self.kd]
            dst = self.W[: self.n_dist]
        for y, d in zip(Y, dst):
            d[:] = np.fft.ifft(y, axis=0)[:c0].reshape(L.world, L.block)

    def finish(self):
        L = self.layout
        c0, c1, c2 = L.counts
        M0, M1, M2 = L.padded
        comps = []
        for w in self.W_recv:
            a = w.reshape(L.world, L.c0loc, L.ks, L.H).transpose(1, 0, 2, 3).reshape(L.c0loc, M1, L.H)
            a = np.fft.ifft(a, axis=1)[:, :c1, :]
            comps.append(np.fft.irfft(a, n=M2, axis=2)[:, :, :c2].reshape(-1))
        phi = comps[0]
        out = {"phi": phi, "S": -self.tau * np.log(np.where(phi > 0, phi, np.nan))}
        if self.grad:
            out["grad"] = [c / phi for c in comps[1:4]]
        if self.sign:
            out["mu"] = -comps[-1] / (4.0 * math.pi)
        return out


class NumpyStreamedSlabExecutor(NumpySlabExecutor):
    """The streamed schedule (slab.run_rank_streamed) on CPU ranks: one V pair
    and one W pair, one input / one component at a time, raw components plus
    an elementwise epilogue."""

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        L = self.layout
        mk = lambda: np.zeros((L.world, L.block), dtype=np.complex128)  # noqa: E731
        self.V_send, self.V_recv, self.W = [mk()], [mk()], [mk()]
        self.W_recv = self.V_send
        self.raw = {}

    def planes_one(self, group, inp, nodes, weights):
        L = self.layout
        c0, c1, c2 = L.counts
        M0, M1, M2 = L.padded
        g = np.zeros(L.c0loc * c1 * c2)
        np.add.at(g, nodes, 1.0 if not group else weights[inp])
        t = np.fft.fft(np.fft.rfft(g.reshape(L.c0loc, c1, c2), n=M2, axis=2), n=M1, axis=1)
        for dest in range(L.world):
            self.V_send[0][dest] = t[:, dest * L.ks:(dest + 1) * L.ks, :].reshape(-1)

    def axis0_one(self, kernel, accumulate=False):
        L = self.layout
        c0, M0 = L.counts[0], L.padded[0]
        k = self.kd[kernel] if kernel < 4 else self.ksg[kernel - 4]
        x = np.fft.fft(self.V_recv[0].reshape(c0, L.ks, L.H), n=M0, axis=0)
        y = np.fft.ifft(k * x, axis=0)[:c0].reshape(L.world, L.block)
        if accumulate:
            self.W[0] += y
        else:
            self.W[0][:] = y

    def finish_raw(self, which):
        L = self.layout
        c0, c1, c2 = L.counts
        M0, M1, M2 = L.padded
        a = self.W_recv[0].reshape(L.world, L.c0loc, L.ks, L.H).transpose(1, 0, 2, 3).reshape(L.c0loc, M1, L.H)
        a = np.fft.ifft(a, axis=1)[:, :c1, :]
        self.raw[which] = np.fft.irfft(a, n=M2, axis=2)[:, :, :c2].reshape(-1).copy()

    def epilogue(self):
        phi = self.raw[0]
        out = {"phi": phi, "S": -self.tau * np.log(np.where(phi > 0, phi, np.nan))}
        if self.grad:
            out["grad"] = [self.raw[j] / phi for j in (1, 2, 3)]
        if self.sign and "mu" in self.raw:
            out["mu"] = -self.raw["mu"] / (4.0 * math.pi)
        return out


class NumpyP2PSlabExecutor(NumpySlabExecutor):
    """The fused peer-to-peer schedule on CPU ranks: every rank's receive arena
    is a shared-memory segment laid out like the CUDA arena ([4 V slots][W
    slots] of [G src][c0/G][ks][H2] complex); planes / axis0 store their blocks
    straight into the owners' arenas, finish reads its own.  The only
    cross-rank operations are the two barriers of slab.run_rank_p2p."""

    NV = 4

    def __init__(self, *args, **kw):
        from multiprocessing import shared_memory

        super().__init__(*args, **kw)
        L = self.layout
        self.n_slots = self.NV + len(self.W)
        self.slot = L.world * L.block
        self.shm = shared_memory.SharedMemory(create=True, size=self.n_slots * self.slot * 16)
        self.name = self.shm.name
        self.peers = None

    def _arena(self, shm):
        L = self.layout
        return np.ndarray((self.n_slots, L.world, L.block), dtype=np.complex128, buffer=shm.buf)

    def connect(self, names):
        from multiprocessing import shared_memory

        self._opened = [self.shm if n == self.name else shared_memory.SharedMemory(name=n) for n in names]
        self.peers = [self._arena(s) for s in self._opened]

    def planes(self, group, nodes, weights):
        super().planes(group, nodes, weights)  # fills V_send[i][dest]
        L = self.layout
        base = 1 if group else 0
        for i in range(3 if group else 1):
            for dest in range(L.world):
                self.peers[dest][base + i, L.rank] = self.V_send[i][dest]

    def axis0(self, group):
        L = self.layout
        own = self.peers[L.rank]
        base = 1 if group else 0
        for i in range(3 if group else 1):
            self.V_recv[i][:] = own[base + i]
        super().axis0(group)  # fills W[j][dest]
        js = [self.n_dist] if group else range(self.n_dist)
        for j in js:
            for dest in range(L.world):
                self.peers[dest][self.NV + j, L.rank] = self.W[j][dest]

    def finish(self):
        own = self.peers[self.layout.rank]
        for j in range(len(self.W_recv)):
            self.W_recv[j][:] = own[self.NV + j]
        return super().finish()

    def close(self):
        for s in self._opened:
            if s is not self.shm:
                s.close()
        self.shm.close()
        self.shm.unlink()
