"""ctypes binding of libeikfld_b200.so (the C ABI in include/eikfld_b200.h).

The library is built in-tree (`python -c "import __graft_entry__ as g; g.build()"`
or `make`).  There is no fallback: if the shared object is missing or no CUDA
device is visible, every entry point raises NativeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from collections import OrderedDict

import numpy as np

from .errors import NativeError, PrecisionError, ValidationError

LIB_PATH = os.environ.get("EIK_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                     "libeikfld_b200.so")

EIK_OK, EIK_EVALIDATION, EIK_EUNDERFLOW, EIK_ECUDA = 0, 1, 2, 3
FIELD_PHI, FIELD_S, FIELD_GRAD, FIELD_HESS, FIELD_WINDING, FIELD_DEGREE = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
HOST_INPUTS, HOST_OUTPUTS, SYNC, CHECK_UNDERFLOW, PROFILE, SLAB_P2P, ASYNC = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40
PASS_NAMES = ("prep", "col", "col_sign", "lines", "row", "col_kernel")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class Inputs(C.Structure):
    _fields_ = [
        ("nodes", C.c_void_p), ("item_offsets", C.c_void_p), ("n_nodes", C.c_int64), ("batch", C.c_int64),
        ("sign_nodes", C.c_void_p), ("n_sign_nodes", C.c_int64), ("sign_weights", C.c_void_p),
    ]


class Outputs(C.Structure):
    _fields_ = [
        ("phi", C.c_void_p), ("S", C.c_void_p), ("grad", C.c_void_p * 3), ("hess", C.c_void_p * 3),
        ("mu", C.c_void_p), ("mask", C.c_void_p), ("underflow", C.c_void_p),
        ("n_underflow", C.c_void_p), ("d_underflow_count", C.c_void_p),
    ]


_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load the shared library once; raise NativeError when it is unavailable."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"CUDA library not built ({LIB_PATH} missing); run `make` or __graft_entry__.build()"
                )
            L = C.CDLL(LIB_PATH)
            L.eik_plan_create.argtypes = [C.c_int, _i64p, C.c_double, C.c_double, C.c_uint32, C.c_int, C.POINTER(C.c_void_p)]
            L.eik_plan_destroy.argtypes = [C.c_void_p]
            L.eik_plan_info.argtypes = [C.c_void_p, _i64p, _i64p, _i64p]
            L.eik_run.argtypes = [C.c_void_p, C.POINTER(Inputs), C.POINTER(Outputs), C.c_uint32, C.c_void_p]
            L.eik_convolve.argtypes = [C.c_int, _i64p, C.c_void_p, C.c_int64, _i64p, C.c_void_p, C.c_void_p,
                                       C.c_uint32, C.c_int, C.c_void_p]
            L.eik_pass_times.argtypes = [C.c_void_p, _f64p, C.c_int]
            L.eik_plan_create_slab.argtypes = [C.c_int, _i64p, C.c_double, C.c_double, C.c_uint32, C.c_int,
                                               C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]
            L.eik_slab_p2p_init.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_void_p,
                                             C.c_void_p, C.c_void_p]
            L.eik_slab_p2p_connect.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.eik_dd_plan_create.argtypes = [C.c_int, _i64p, C.c_double, C.c_double, C.c_uint32, C.c_int,
                                              C.POINTER(C.c_void_p)]
            L.eik_dd_plan_destroy.argtypes = [C.c_void_p]
            L.eik_dd_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_uint32, C.c_void_p]
            L.eik_plan_create_sweep.argtypes = [C.c_int, _i64p, C.c_double, _f64p, C.c_int, C.c_int,
                                                C.POINTER(C.c_void_p)]
            L.eik_run_sweep.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_uint32,
                                        C.c_void_p]
            L.eik_classify.argtypes = [C.c_int, _i64p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                       C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_int,
                                       C.c_void_p]
            L.eik_slab_planes.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                          C.c_int64, C.c_void_p, C.c_uint32, C.c_void_p]
            L.eik_slab_axis0.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                         C.c_uint32, C.c_void_p]
            L.eik_slab_finish.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(Outputs),
                                          C.c_uint32, C.c_void_p]
            L.eik_slab_fill.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
            L.eik_fftn.argtypes = [C.c_int, _i64p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_uint32, C.c_int,
                                   C.c_void_p]
            L.eik_fft_pair.argtypes = [C.c_int, _i64p, C.c_void_p, _i64p, C.c_void_p, _i64p, C.c_void_p, C.c_void_p,
                                       C.c_uint32, C.c_int, C.c_void_p]
            L.eik_ifft_window.argtypes = [C.c_int, _i64p, C.c_void_p, C.c_void_p, _i64p, _i64p, C.c_void_p,
                                          C.c_void_p, C.c_uint32, C.c_int, C.c_void_p]
            L.eik_cmul.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p]
            L.eik_slab_planes_one.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                              C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
            L.eik_slab_axis0_one.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                             C.c_int, C.c_void_p]
            L.eik_slab_finish_raw.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
            L.eik_slab_epilogue.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(Outputs),
                                            C.c_void_p]
            L.eik_last_error.restype = C.c_char_p
            for name in ("eik_slab_planes_one", "eik_slab_axis0_one", "eik_slab_finish_raw", "eik_slab_epilogue"):
                getattr(L, name).restype = C.c_int
            for name in ("eik_plan_create", "eik_plan_destroy", "eik_plan_info", "eik_run", "eik_convolve",
                         "eik_version", "eik_pass_times", "eik_plan_create_slab", "eik_slab_planes",
                         "eik_slab_axis0", "eik_slab_finish", "eik_plan_create_sweep", "eik_run_sweep",
                         "eik_classify", "eik_slab_p2p_init", "eik_slab_p2p_connect", "eik_dd_plan_create",
                         "eik_dd_plan_destroy", "eik_dd_run", "eik_slab_fill", "eik_fftn", "eik_fft_pair",
                         "eik_ifft_window", "eik_cmul"):
                getattr(L, name).restype = C.c_int
            _lib = L
        return _lib


def exported_symbols():
    return ["eik_plan_create", "eik_plan_create_slab", "eik_plan_destroy", "eik_plan_info", "eik_run",
            "eik_convolve", "eik_slab_planes", "eik_slab_axis0", "eik_slab_finish", "eik_pass_times",
            "eik_plan_create_sweep", "eik_run_sweep", "eik_classify", "eik_slab_p2p_init", "eik_slab_p2p_connect",
            "eik_dd_plan_create", "eik_dd_plan_destroy", "eik_dd_run", "eik_slab_fill",
            "eik_slab_planes_one", "eik_slab_axis0_one", "eik_slab_finish_raw", "eik_slab_epilogue",
            "eik_fftn", "eik_fft_pair", "eik_ifft_window", "eik_cmul",
            "eik_last_error", "eik_version"]


def check(rc: int):
    if rc == EIK_OK:
        return
    msg = lib().eik_last_error().decode(errors="replace")
    if rc == EIK_EVALIDATION:
        raise ValidationError(msg)
    if rc == EIK_EUNDERFLOW:
        raise PrecisionError(msg)
    raise NativeError(msg)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor (device or host)


class Plan:
    """Owns one eik_plan: geometry, twiddles and cached kernel spectra on one device."""

    def __init__(self, dim, counts, spacing, tau, fields, device=0, k1_slab=None):
        self.dim = int(dim)
        self.counts = tuple(int(c) for c in counts)
        self.spacing = float(spacing)
        self.tau = float(tau)
        self.fields = int(fields)
        self.device = int(device)
        self.N = int(np.prod(self.counts))
        h = C.c_void_p()
        cnt = (C.c_int64 * 3)(*self.counts, *([1] * (3 - len(self.counts))))
        if k1_slab is None:
            check(lib().eik_plan_create(self.dim, cnt, self.spacing, self.tau, self.fields, self.device, C.byref(h)))
        else:
            check(lib().eik_plan_create_slab(self.dim, cnt, self.spacing, self.tau, self.fields, self.device,
                                             int(k1_slab[0]), int(k1_slab[1]), C.byref(h)))
        self._h = h
        self._lock = threading.Lock()

    def info(self):
        pad = (C.c_int64 * 3)()
        lines = C.c_int64()
        nbytes = C.c_int64()
        check(lib().eik_plan_info(self._h, pad, C.byref(lines), C.byref(nbytes)))
        return {"padded": tuple(pad), "lines": lines.value, "device_bytes": nbytes.value}

    # -- slab-decomposed 3-D passes (device tensors; see include/eikfld_b200.h)
    def slab_planes(self, group, nodes, weights, c0_local, ks, v_out=None, stream=None, p2p=False):
        v_out = v_out or []
        arr = (C.c_void_p * 3)(*[_ptr(t) for t in v_out], *([None] * (3 - len(v_out))))
        check(lib().eik_slab_planes(self._h, int(group), _ptr(nodes), int(nodes.shape[0]),
                                    _ptr(weights), int(c0_local), int(ks), arr, SLAB_P2P if p2p else 0, stream))

    def slab_axis0(self, group, v_in, k1_begin, ks, w_out, stream=None, p2p=False):
        v_in, w_out = v_in or [], w_out or []
        vi = (C.c_void_p * 3)(*[_ptr(t) for t in v_in], *([None] * (3 - len(v_in))))
        wo = (C.c_void_p * 8)(*[_ptr(t) for t in w_out], *([None] * (8 - len(w_out))))
        check(lib().eik_slab_axis0(self._h, int(group), vi, int(k1_begin), int(ks), wo, SLAB_P2P if p2p else 0,
                                   stream))

    def slab_p2p_init(self, world, rank, c0_local, ks):
        """Allocate the peer-to-peer exchange arena -> (device pointer, bytes, 64-byte IPC handle)."""
        arena = C.c_void_p()
        nbytes = C.c_int64()
        handle = (C.c_char * 64)()
        check(lib().eik_slab_p2p_init(self._h, int(world), int(rank), int(c0_local), int(ks), C.byref(arena),
                                      C.byref(nbytes), handle))
        return arena.value, nbytes.value, bytes(handle)

    def slab_p2p_connect(self, peer_arenas=None, ipc_handles=None):
        """Peers by device pointer (same process) or by IPC handle (list of 64-byte strings)."""
        pa = None
        if peer_arenas is not None:
            pa = (C.c_void_p * len(peer_arenas))(*peer_arenas)
        hb = None
        if ipc_handles is not None:
            hb = C.create_string_buffer(b"".join(ipc_handles), 64 * len(ipc_handles))
        check(lib().eik_slab_p2p_connect(self._h, pa, hb))

    def slab_finish(self, w, c0_local, ks, *, S=None, grad=(None, None, None), mu=None, mask=None,
                    underflow=None, d_count=None, stream=None, p2p=False):
        w = w or []
        wa = (C.c_void_p * 8)(*[_ptr(t) for t in w], *([None] * (8 - len(w))))
        out = Outputs()
        out.S, out.mu, out.mask, out.underflow = (_ptr(x) for x in (S, mu, mask, underflow))
        for d in range(3):
            out.grad[d] = _ptr(grad[d]) if d < len(grad) else None
        out.d_underflow_count = _ptr(d_count)
        check(lib().eik_slab_finish(self._h, wa, int(c0_local), int(ks), C.byref(out), SLAB_P2P if p2p else 0,
                                    stream))

    # -- streamed slab schedule: one input / one component at a time
    def slab_planes_one(self, group, inp, nodes, weights, c0_local, ks, v_out, stream=None):
        check(lib().eik_slab_planes_one(self._h, int(group), int(inp), _ptr(nodes), int(nodes.shape[0]),
                                        _ptr(weights), int(c0_local), int(ks), _ptr(v_out), stream))

    def slab_axis0_one(self, kernel, v_in, k1_begin, ks, w_out, accumulate=False, stream=None):
        check(lib().eik_slab_axis0_one(self._h, int(kernel), _ptr(v_in), int(k1_begin), int(ks), _ptr(w_out),
                                       1 if accumulate else 0, stream))

    def slab_finish_raw(self, w, c0_local, ks, raw_out, stream=None):
        check(lib().eik_slab_finish_raw(self._h, _ptr(w), int(c0_local), int(ks), _ptr(raw_out), stream))

    def slab_epilogue(self, n_local, phi_raw, mu_raw, *, S=None, grad=(None, None, None), mu=None, mask=None,
                      underflow=None, stream=None):
        out = Outputs()
        out.S, out.mu, out.mask, out.underflow = (_ptr(x) for x in (S, mu, mask, underflow))
        for d in range(3):
            out.grad[d] = _ptr(grad[d]) if d < len(grad) else None
        check(lib().eik_slab_epilogue(self._h, int(n_local), _ptr(phi_raw), _ptr(mu_raw), C.byref(out), stream))

    def slab_fill(self, ext_nodes, e0, e1, own0, c0_local, mask_ext, mask_own, stream=None):
        check(lib().eik_slab_fill(self._h, _ptr(ext_nodes), int(ext_nodes.shape[0]), int(e0), int(e1), int(own0),
                                  int(c0_local), _ptr(mask_ext), _ptr(mask_own), stream))

    def pass_times(self):
        """Device ms per pass of the last profiled run ({name: ms}, absent passes omitted)."""
        ms = (C.c_double * len(PASS_NAMES))()
        check(lib().eik_pass_times(self._h, ms, len(PASS_NAMES)))
        return {n: v for n, v in zip(PASS_NAMES, ms) if v >= 0}

    def close(self):
        """Destroy the native plan; waits for a run in progress on another thread."""
        h = getattr(self, "_h", None)
        if C is None or h is None:  # interpreter shutdown: module globals already gone
            return
        lock = getattr(self, "_lock", None)
        if lock is not None:
            lock.acquire()
        try:
            h = self._h
            if h.value:
                self._h = C.c_void_p()
                try:
                    lib().eik_plan_destroy(h)
                except Exception:  # interpreter shutdown: the process releases the device anyway
                    pass
        finally:
            if lock is not None:
                lock.release()

    __del__ = close

    def run(self, nodes=None, item_offsets=None, batch=1, sign_nodes=None, sign_weights=None, *,
            phi=None, S=None, grad=(None, None, None), hess=(None, None, None), mu=None, mask=None,
            underflow=None, count=False, check_underflow=False, host=True, stream=None, profile=False,
            wait=True):
        """Run the hot path.  Arrays are numpy (host=True) or torch CUDA tensors (host=False).

        host=True, wait=False queues the run and returns (EIK_ASYNC): outputs are
        complete once `stream` is; the next run's column passes overlap this D2H.
        """
        inp = Inputs()
        keep = []
        if nodes is not None:
            inp.nodes = _ptr(nodes)
            inp.n_nodes = int(nodes.shape[0])
            keep.append(nodes)
        if item_offsets is not None:
            inp.item_offsets = _ptr(item_offsets)
            keep.append(item_offsets)
        inp.batch = int(batch)
        if sign_nodes is not None:
            inp.sign_nodes = _ptr(sign_nodes)
            inp.n_sign_nodes = int(sign_nodes.shape[0])
            inp.sign_weights = _ptr(sign_weights)
            keep += [sign_nodes, sign_weights]
        out = Outputs()
        out.phi, out.S, out.mu, out.mask, out.underflow = (_ptr(x) for x in (phi, S, mu, mask, underflow))
        for d in range(3):
            out.grad[d] = _ptr(grad[d]) if d < len(grad) else None
            out.hess[d] = _ptr(hess[d]) if d < len(hess) else None
        n_uf = C.c_int64(-1)
        if count or check_underflow:
            out.n_underflow = C.addressof(n_uf)
        flags = (HOST_INPUTS | HOST_OUTPUTS) if host else 0
        if check_underflow:
            flags |= CHECK_UNDERFLOW
        if profile:
            flags |= PROFILE
        if host and not wait:
            flags |= ASYNC
        with self._lock:
            rc = lib().eik_run(self._h, C.byref(inp), C.byref(out), flags, stream)
        check(rc)
        return n_uf.value


_PLANS: "OrderedDict[tuple, Plan]" = OrderedDict()
_PLANS_LOCK = threading.Lock()
_MAX_PLANS = 8


def get_plan(grid, tau, fields, device=0) -> Plan:
    """Plan cache keyed by (device, counts, spacing, tau, fields) — the analogue
    of the reference's plan cache (R/convolution.py:70-71,105-112)."""
    key = (device, tuple(grid.counts), float(grid.spacing), float(tau), int(fields))
    with _PLANS_LOCK:
        p = _PLANS.get(key)
        if p is not None:
            _PLANS.move_to_end(key)
            return p
    p = Plan(len(grid.counts), grid.counts, grid.spacing, tau, fields, device)
    with _PLANS_LOCK:
        _PLANS[key] = p
        while len(_PLANS) > _MAX_PLANS:
            # dropped, not closed: a thread may still be running on it; the
            # plan is destroyed by __del__ once the last reference is gone
            _PLANS.popitem(last=False)
    return p


def clear_plans():
    with _PLANS_LOCK:
        for p in _PLANS.values():
            p.close()
        _PLANS.clear()


def convolve(counts, kernels, field, device=0):
    """Host-in/host-out linear convolution of stacked centred kernels with a dense field."""
    counts = tuple(int(c) for c in counts)
    kernels = np.ascontiguousarray(kernels, dtype=np.float64)
    field = np.ascontiguousarray(field, dtype=np.float64).reshape(-1)
    n = kernels.shape[0]
    kshape = kernels.shape[1:]
    out = np.empty((n, int(np.prod(counts))), dtype=np.float64)
    cnt = (C.c_int64 * 3)(*counts, *([1] * (3 - len(counts))))
    ks = (C.c_int64 * 3)(*kshape, *([1] * (3 - len(kshape))))
    check(lib().eik_convolve(len(counts), cnt, kernels.ctypes.data, n, ks, field.ctypes.data, out.ctypes.data,
                             HOST_INPUTS | HOST_OUTPUTS, device, None))
    return out


class DDOutputs(C.Structure):
    _fields_ = [("phi_hi", C.c_void_p), ("phi_lo", C.c_void_p), ("S", C.c_void_p), ("grad", C.c_void_p * 3),
                ("hess", C.c_void_p * 3), ("underflow", C.c_void_p), ("n_underflow", C.c_void_p)]


class DDPlan:
    """Double-double (~106-bit) convolution plan: the big-float path of the
    reference (R/convolution.py:67-143) with p = 106."""

    def __init__(self, dim, counts, spacing, tau, fields, device=0):
        self.dim = int(dim)
        self.counts = tuple(int(c) for c in counts)
        self.N = int(np.prod(self.counts))
        h = C.c_void_p()
        cnt = (C.c_int64 * 3)(*self.counts, *([1] * (3 - len(self.counts))))
        check(lib().eik_dd_plan_create(self.dim, cnt, float(spacing), float(tau), int(fields), int(device),
                                       C.byref(h)))
        self._h = h
        self._lock = threading.Lock()

    def run(self, nodes, *, phi_hi=None, phi_lo=None, S=None, grad=(None, None, None), hess=(None, None, None),
            underflow=None, check_underflow=False):
        """Host arrays in and out; returns the number of nodes with phi <= 0."""
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        o = DDOutputs()
        o.phi_hi, o.phi_lo, o.S, o.underflow = (_ptr(x) for x in (phi_hi, phi_lo, S, underflow))
        for d in range(3):
            o.grad[d] = _ptr(grad[d]) if d < len(grad) else None
            o.hess[d] = _ptr(hess[d]) if d < len(hess) else None
        n_uf = C.c_int64(-1)
        o.n_underflow = C.addressof(n_uf)
        flags = HOST_INPUTS | HOST_OUTPUTS | SYNC | (CHECK_UNDERFLOW if check_underflow else 0)
        with self._lock:
            rc = lib().eik_dd_run(self._h, _ptr(nodes), int(nodes.shape[0]), C.byref(o), flags, None)
        check(rc)
        return n_uf.value

    def close(self):
        h = getattr(self, "_h", None)
        if C is None or h is None:  # interpreter shutdown: module globals already gone
            return
        lock = getattr(self, "_lock", None)
        if lock is not None:
            lock.acquire()
        try:
            h = self._h
            if h.value:
                self._h = C.c_void_p()
                try:
                    lib().eik_dd_plan_destroy(h)
                except Exception:
                    pass
        finally:
            if lock is not None:
                lock.release()

    __del__ = close


_DD_PLANS: "OrderedDict" = OrderedDict()


def get_dd_plan(grid, tau, fields, device=0) -> DDPlan:
    key = (device, tuple(grid.counts), float(grid.spacing), float(tau), int(fields))
    with _PLANS_LOCK:
        p = _DD_PLANS.get(key)
        if p is not None:
            _DD_PLANS.move_to_end(key)
            return p
    p = DDPlan(len(grid.counts), grid.counts, grid.spacing, tau, fields, device)
    with _PLANS_LOCK:
        _DD_PLANS[key] = p
        while len(_DD_PLANS) > 2:  # DD plans are large (32 B per padded point per kernel)
            _DD_PLANS.popitem(last=False)  # freed by __del__ once no thread holds it
    return p


class SweepPlan(Plan):
    """tau-sweep plan: exp spectra for several tau values over one grid (1-D / 2-D)."""

    def __init__(self, dim, counts, spacing, taus, device=0):  # noqa: super-init replaced
        self.dim = int(dim)
        self.counts = tuple(int(c) for c in counts)
        self.spacing = float(spacing)
        self.taus = [float(t) for t in taus]
        self.device = int(device)
        self.N = int(np.prod(self.counts))
        h = C.c_void_p()
        cnt = (C.c_int64 * 3)(*self.counts, *([1] * (3 - len(self.counts))))
        tt = (C.c_double * len(self.taus))(*self.taus)
        check(lib().eik_plan_create_sweep(self.dim, cnt, self.spacing, tt, len(self.taus), self.device, C.byref(h)))
        self._h = h
        self._lock = threading.Lock()

    def run_sweep(self, nodes, outs, host=True, stream=None):
        arr = (C.c_void_p * len(outs))(*[_ptr(o) for o in outs])
        n_uf = C.c_int64(-1)
        flags = (HOST_INPUTS | HOST_OUTPUTS) if host else SYNC
        with self._lock:
            rc = lib().eik_run_sweep(self._h, _ptr(nodes), int(nodes.shape[0]), arr, C.addressof(n_uf), flags, stream)
        check(rc)
        return n_uf.value


def classify(counts, mu, flagged, mode, threshold=None, S=None, device=0):
    """GPU interior mask (float64 0/1) and, with S, the signed distance; host arrays."""
    counts = tuple(int(c) for c in counts)
    N = int(np.prod(counts))
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    fl = None if flagged is None else np.ascontiguousarray(flagged, dtype=np.int64)
    mask = np.empty(N)
    sd = None
    if S is not None:
        S = np.ascontiguousarray(S, dtype=np.float64)
        sd = np.empty(N)
    cnt = (C.c_int64 * 3)(*counts, *([1] * (3 - len(counts))))
    check(lib().eik_classify(len(counts), cnt, mu.ctypes.data, None if fl is None else fl.ctypes.data,
                             0 if fl is None else fl.size, int(mode), threshold is not None,
                             0.0 if threshold is None else float(threshold), mask.ctypes.data,
                             None if S is None else S.ctypes.data, None if sd is None else sd.ctypes.data,
                             HOST_INPUTS | HOST_OUTPUTS, device, None))
    return mask, sd


# -- engine-level spectral API (R/convolution.py:164-313) -----------------------

def _dims(shape):
    return (C.c_int64 * max(1, len(shape)))(*[int(x) for x in shape])


def fftn(array, inverse=False, device=0):
    """Forward (unnormalised) or inverse (1/P) DFT over every axis; host arrays, complex128 out."""
    arr = np.asarray(array)
    real = not np.iscomplexobj(arr)
    src = np.ascontiguousarray(arr, dtype=np.float64 if real else np.complex128)
    out = np.empty(src.shape, dtype=np.complex128)
    check(lib().eik_fftn(src.ndim, _dims(src.shape), src.ctypes.data, int(real), out.ctypes.data, int(bool(inverse)),
                         HOST_INPUTS | HOST_OUTPUTS, device, None))
    return out


def fft_pair(pshape, a, ashape, b, bshape, device=0):
    """forward_pair: spectra of two real arrays zero-padded to pshape (one complex transform)."""
    a = None if a is None else np.ascontiguousarray(a, dtype=np.float64)
    b = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
    ah = np.empty(tuple(pshape), dtype=np.complex128)
    bh = np.empty(tuple(pshape), dtype=np.complex128)
    check(lib().eik_fft_pair(len(pshape), _dims(pshape), None if a is None else a.ctypes.data, _dims(ashape),
                             None if b is None else b.ctypes.data, _dims(bshape), ah.ctypes.data, bh.ctypes.data,
                             HOST_INPUTS | HOST_OUTPUTS, device, None))
    return ah, bh


def ifft_window(hat_a, hat_b, start, counts, want_imag, device=0):
    """Inverse of hat_a (+ i hat_b) restricted to the window [start, start + counts): (real, imag|None)."""
    ha = np.ascontiguousarray(hat_a, dtype=np.complex128)
    hb = None if hat_b is None else np.ascontiguousarray(hat_b, dtype=np.complex128)
    if hb is not None and hb.shape != ha.shape:
        raise ValidationError("spectra of different shapes")
    re = np.empty(tuple(counts))
    im = np.empty(tuple(counts)) if want_imag else None
    check(lib().eik_ifft_window(ha.ndim, _dims(ha.shape), ha.ctypes.data, None if hb is None else hb.ctypes.data,
                                _dims(start), _dims(counts), re.ctypes.data, None if im is None else im.ctypes.data,
                                HOST_INPUTS | HOST_OUTPUTS, device, None))
    return re, im


def cmul(a, b, device=0):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    if a.shape != b.shape:
        a, b = np.broadcast_arrays(a, b)
        a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    out = np.empty(a.shape, dtype=np.complex128)
    check(lib().eik_cmul(a.size, a.ctypes.data, b.ctypes.data, out.ctypes.data, HOST_INPUTS | HOST_OUTPUTS, device,
                         None))
    return out
