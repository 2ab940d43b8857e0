#!/usr/bin/env python
"""Benchmark of the B200 FFT-convolution distance transform (contract: see DESIGN.md §Measurement).

Default workload = BASELINE.json configs[1] ("C2"): signed distance + Hessian
on a 2048^2 grid — S, grad S, (S_xx, S_yy, S_xy), winding number mu and the
interior mask, tau = 0.5, float64 — from the seeded synthetic star curve
(workloads.c2).  Metric: grid points per second (whole job, all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C1..C5]

One process per GPU (torchrun for N > 1).  C1-C3 do not shard: N ranks run N
independent replicas ("weak").  C5 shards its 512 items across ranks with no
communication ("strong").  `--impl reference` times the CPU oracle
(oracle/eikfld_oracle.py, a bit-exact restatement of the reference's float64
path) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

CONFIG_TEXT = {
    "C1": "2D 256^2, K=2000 random nodes, tau=0.5: S + grad S",
    "C2": "2D 2048^2 star curve (16384 vertices, 5908 distinct nodes), tau=0.5: S + grad S + Hessian + winding sign",
    "C3": "3D 256^3, 16 ellipsoids x 12500 points (105389 distinct nodes), tau=0.5: S + grad S",
    "C5": "batched 2D: 512 items x 512^2, K=1000 nodes each, tau=0.5: S + grad S per item",
    "TS": "tau sweep (SURVEY 8(f) rank 1): C2's 2048^2 delta_Y, S for 9 taus 0.5..4.5 from one transform "
          "(metric counts grid points x taus)",
    "C4": "3D 1024^3 perturbed icosphere (501,762 vertices, vector-area normals), tau=0.75: S + grad S + degree sign; "
          "slab-decomposed, exchange fused into the passes as NVLink peer stores (--exchange nccl: NCCL "
          "all-to-all); 1 GPU: eik_run's streamed schedule; 2 GPUs: streamed slab schedule over NCCL",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIG_TEXT))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--items", type=int, default=512, help="C5 batch size (whole job)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="C4 slab exchange: fused peer stores (p2p) or NCCL all_to_all_single")
    ap.add_argument("--c4-size", type=int, default=0,
                    help="C4 grid edge (default 1024 at every rank count; smaller grids scale the surface)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no device work: launch the ranks (gloo), build each rank's shard and print the line "
                         "skeleton (tests the multi-rank plumbing on CPU)")
    return ap.parse_args()


# ---------------------------------------------------------------- ranks


def spawn_ranks(a):
    """`--gpus N` outside torchrun: re-launch this script with N local ranks
    (torch.distributed.run, rendezvous on 127.0.0.1), return its exit code."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def rank_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init_ranks(world, local, cpu_only=False):
    """(dist | None, device index, oversubscribed).  NCCL when every rank has its
    own GPU; gloo on CPU (dry runs, tests) or when ranks share a device (NCCL
    cannot place two ranks on one GPU; such a run is a functional check only)."""
    if world <= 1:
        return None, local, False
    import torch
    import torch.distributed as dist

    ndev = 0 if cpu_only or not torch.cuda.is_available() else torch.cuda.device_count()
    over = ndev < world
    if ndev and not over:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    return dist, (local % ndev if ndev else local), over


def reduce_max(dist, value, dev=None):
    """Max over ranks (device tensor for NCCL, host tensor for gloo)."""
    if dist is None:
        return value
    import torch

    on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_items(items, rank, world):
    """C5: rank r takes items [r*per, (r+1)*per), per = items // world (no data-path collective)."""
    per = items // world
    return rank * per, per


# ---------------------------------------------------------------- workloads


def build_workload(cfg, seed, rank=0, world=1, items=512):
    from paper_1112_3010_b200 import workloads as wl
    from paper_1112_3010_b200.sign import FluxData, TangentData

    if cfg == "C1":
        d = wl.c1(seed)
        return dict(grid=d["grid"], tau=d["tau"], nodes=[d["points"].distinct_nodes()], grad=True)
    if cfg == "C2":
        d = wl.c2(seed)
        td = TangentData.build(d["curve"], d["grid"])
        return dict(grid=d["grid"], tau=d["tau"], nodes=[d["points"].distinct_nodes()], grad=True, hess=True,
                    sign=(td.nodes, np.ascontiguousarray(td.weights)), curve=d["curve"])
    if cfg == "C3":
        d = wl.c3(seed)
        return dict(grid=d["grid"], tau=d["tau"], nodes=[d["points"].distinct_nodes()], grad=True)
    if cfg == "C5":
        first, per = shard_items(items, rank, world)
        d = wl.c5(seed, items=per, first=first)
        return dict(grid=d["grid"], tau=d["tau"], nodes=[p.distinct_nodes() for p in d["items"]], grad=True,
                    items_total=per * world)
    raise ValueError(cfg)


SURVEY_BYTES_PER_POINT = {"C1": 264, "C2": 696, "C3": 768, "C4": 1640, "C5": 264}


def algorithmic_bytes(plan_info, w, batch):
    """Compulsory HBM bytes per launch of each pass (DESIGN.md §Roofline model).

    2-D, c0 x c1 grid, H = M1/2+1 spectral columns, kernel spectra folded to
    (M0/2+1) x H doubles:  col = n_k*8*(M0/2+1)*H + n_c*16*c0*H ;
    row = n_c*16*c0*H + (8*n_f64_out + n_u8_out)*N.
    """
    grid = w["grid"]
    if len(grid.counts) == 3:
        return algorithmic_bytes_3d(plan_info, w, batch)
    if len(grid.counts) != 2:
        return {}
    c0, c1 = grid.counts
    M0 = plan_info["padded"][0]
    H = plan_info["lines"]
    dim = 2
    n_dist = 1 + (dim if w.get("grad") else 0) + (3 if w.get("hess") else 0)
    ks = (M0 // 2 + 1) * H * 8
    out = {"col": batch * n_dist * 16 * c0 * H + n_dist * ks}
    n_c = n_dist
    if w.get("sign") is not None:
        out["col_sign"] = 16 * c0 * H + 2 * ks
        n_c += 1
    n_f64 = 1 + (dim if w.get("grad") else 0) + (3 if w.get("hess") else 0) + (1 if w.get("sign") is not None else 0)
    n_u8 = 1 if w.get("sign") is not None else 0
    out["row"] = batch * (n_c * 16 * c0 * H + (8 * n_f64 + n_u8) * c0 * c1)
    return out


def c4_step_bytes(counts, padded):
    """Compulsory HBM bytes of one fused C4 step (S + grad S + degree sign), 3-D pass model of
    algorithmic_bytes_3d extended by the sign group: three flux inputs (T and V round trips,
    one folded spectrum each), one summed component through the lines and row passes, mu and
    the mask.  The streamed one-GPU schedule moves more (it repeats the axis-0 forward per
    component and accumulates the sign component in HBM); this is the bound, not its traffic."""
    c0, c1, c2 = counts
    M0, M1, M2 = padded[:3]
    H = M2 // 2 + 1
    ks = (M0 // 2 + 1) * (M1 // 2 + 1) * H * 8
    plane = 16 * c0 * M1 * H
    slab = 16 * c0 * c1 * H
    N = c0 * c1 * c2
    dist = (2 * slab + 2 * plane) + 4 * (ks + 2 * plane + 2 * slab + 8 * N)
    sign = 3 * (2 * slab + 2 * plane + ks) + (2 * plane + 2 * slab) + 9 * N
    return dist + sign


def algorithmic_bytes_3d(plan_info, w, batch):
    """3-D pass model (c0 x c1 x c2 grid, M = 2c, H = M2/2+1).

    col   = impulse rows T (16*c0*c1*H written + read) + V (16*c0*M1*H written
            by the axis-1 forward, read by the axis-0 pass) + kernel spectra
            n_k*8*(M0/2+1)*(M1/2+1)*H + components n_c*16*c0*M1*H written;
    lines = n_c*16*c0*M1*H read + n_c*16*c0*c1*H written (axis-1 inverse);
    row   = n_c*16*c0*c1*H read + (8*n_f64_out + n_u8_out)*N written.
    """
    c0, c1, c2 = w["grid"].counts
    M0, M1, M2 = plan_info["padded"][:3]
    H = M2 // 2 + 1
    n_c = 1 + (3 if w.get("grad") else 0)
    ks = (M0 // 2 + 1) * (M1 // 2 + 1) * H * 8  # stored folded along every axis
    plane = 16 * c0 * M1 * H
    slab = 16 * c0 * c1 * H
    out = {"col": batch * (2 * slab + 2 * plane + n_c * plane) + n_c * ks,
           "lines": batch * n_c * (plane + slab),
           "row": batch * (n_c * slab + 8 * n_c * c0 * c1 * c2)}
    return out


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.

    NVML is polled in-process every ~1 ms (a C2 timed region is ~15 ms, far too
    short for nvidia-smi's 100 ms loop); falls back to nvidia-smi if NVML is absent.
    """

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.nv, self.h = nv, h
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    self.sample()
                    time.sleep(0.001)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            time.sleep(0.005)  # at least one sample before the region starts
        except Exception:
            self.nv = None
        return self

    def sample(self):
        try:
            nv, h = self.nv, self.h
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((sm, self.max_mhz, rs))
        except Exception:
            pass

    def __exit__(self, *exc):
        # one synchronous sample at the end of the region as well (the poller
        # can be starved of the GIL while the timed loop enqueues)
        if self.nv is not None:
            self.sample()
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "none"}
        sm = [x[0] for x in self.samples]
        reasons = set()
        for _, _, rs in self.samples:
            for name, const in self.REASONS.items():
                if rs & getattr(self.nv, const, 0):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(self.samples[0][1]), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml"}


# ---------------------------------------------------------------- CPU side


def oracle_step(w):
    """One pass of the reference algorithm (oracle port) over the workload; returns grid points done."""
    import eikfld_oracle as orc

    grid = w["grid"]
    pts = 0
    for nodes in w["nodes"]:
        orc.phi_unchecked(nodes, grid.counts, grid.spacing, w["tau"])  # s_fft's convolution
        if w.get("hess"):
            orc.hessian_2d_unchecked(nodes, grid.counts, grid.spacing, w["tau"])  # ratio batch incl. gradient
        elif w.get("grad"):
            orc.gradient_unchecked(nodes, grid.counts, grid.spacing, w["tau"])
        pts += grid.num_nodes
    if w.get("curve") is not None:
        mu, flagged = orc.winding_field(w["curve"].vertices, grid.origin, grid.spacing, grid.counts)
        orc.classify(mu, flagged, grid.counts, "winding2d")  # the mask, flagged nodes filled (R/sign.py:166-198)
    return pts


def cpu_time(w, steps, warmup, budget_s=None, workers=None):
    import scipy.fft as sfft

    sys.path.insert(0, os.path.join(REPO, "oracle"))
    cores = workers or os.cpu_count() or 1
    with sfft.set_workers(cores):
        for _ in range(warmup):
            oracle_step(w)
        t0 = time.perf_counter()
        pts = 0
        done = 0
        for _ in range(steps):
            pts += oracle_step(w)
            done += 1
            if budget_s is not None and time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
    return pts / dt, dt / done, done, cores


# ---------------------------------------------------------------- GPU side


def parallelism(cfg, world, over=False):
    p = {"C5": f"batch-shard x{world} (no data-path collective)", "C4": f"slab x{world}"}.get(
        cfg, f"replicas x{world} (the grid does not shard)")
    return p + (" [ranks share one device: functional check, not a scaling number]" if over else "")


def dry_run(a):
    """Rank plumbing without device work: every rank builds its shard; rank 0 prints the gathered layout."""
    rank, world, local = rank_env()
    dist, _, _ = init_ranks(world, local, cpu_only=True)
    if a.config in ("C1", "C2", "C3", "C5"):
        w = build_workload(a.config, a.seed, rank, world, a.items)
        first = shard_items(a.items, rank, world)[0] if a.config == "C5" else 0
        mine = {"rank": rank, "first_item": first, "items": len(w["nodes"]),
                "nodes": int(sum(len(n) for n in w["nodes"])), "grid_points": len(w["nodes"]) * w["grid"].num_nodes}
    else:
        mine = {"rank": rank}
    shards = [mine]
    if dist:
        shards = [None] * world
        dist.all_gather_object(shards, mine)
    slowest = reduce_max(dist, float(rank))
    if rank == 0:
        pts = sum(x.get("grid_points", 0) for x in shards)
        print(json.dumps({"metric": "grid points/sec (S+grad S+sign)", "value": None, "unit": "grid_points/s",
                          "n_gpus": world, "dry_run": True, "steps": 0, "warmup": 0,
                          "scaling": "strong" if a.config in ("C4", "C5") else "weak",
                          "config": {"workload": a.config, "desc": CONFIG_TEXT[a.config],
                                     "parallelism": parallelism(a.config, world)},
                          "grid_points_per_step_job": pts, "shards": shards, "max_over_ranks_check": slowest}))
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(a)
    if a.dry_run:
        return dry_run(a)
    if a.config == "C4" and a.impl == "b200":
        return bench_c4(a)
    if a.config == "TS":
        return bench_sweep(a)
    rank, world, local = rank_env()
    sys.path.insert(0, os.path.join(REPO, "oracle"))

    if a.impl == "reference":
        if rank != 0:
            return 0
        if a.config == "C4":
            print(json.dumps({"impl": "reference", "unavailable": "the reference algorithm pads 1024^3 to 3072^3 "
                              "(464 GB per complex array) and caps FFTs at 2^31 elements (R/convolution.py:180-184)"}))
            return 0
        w = build_workload(a.config, a.seed, 0, 1, min(a.items, 8))
        if a.config == "C5":
            w["nodes"] = w["nodes"][:8]
        # CPU has no warm-up effects worth W full steps of a ~10 s pipeline; one is run
        val, sec, done, cores = cpu_time(w, a.steps, min(a.warmup, 1), budget_s=240.0)
        # the reference as shipped: scipy.fft's default single worker, one step
        # (the public calls raise PrecisionError on C2/C3/C5 only after all
        # their transforms ran, R/convolution.py:378-388, so the unchecked
        # pipeline takes the same time)
        v1, sec1, _, _ = cpu_time(w, 1, 0, workers=1)
        line = {
            "metric": "grid points/sec (S+grad S+sign)", "value": val, "unit": "grid_points/s", "n_gpus": a.gpus,
            "steps": done, "warmup": min(a.warmup, 1), "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak" if a.config != "C5" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": a.config, "desc": CONFIG_TEXT[a.config]},
            "cpu_baseline": {"value": val, "unit": "grid_points/s", "cores": cores, "kind": "port",
                             "sample": f"{done} step(s) of the oracle pipeline on {a.config}"
                                       + (" (8 of 512 items per step)" if a.config == "C5" else "")
                                       + f", scipy.fft workers={cores}"},
            "e2e": {"value": val, "unit": "grid_points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "as_shipped": {"value": v1, "unit": "grid_points/s", "cores": 1, "ms_per_step": sec1 * 1e3,
                           "sample": "1 step, scipy.fft workers=1 (the reference's default)"},
        }
        print(json.dumps(line))
        return 0

    import torch

    dist, local, over = init_ranks(world, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1112_3010_b200 import _native
    from paper_1112_3010_b200.engine import field_bits

    w = build_workload(a.config, a.seed, rank, world, a.items)
    grid = w["grid"]
    dim = len(grid.counts)
    t_plan = time.perf_counter()
    plan = _native.Plan(dim, grid.counts, grid.spacing, w["tau"],
                        field_bits(dim, w.get("grad", False), w.get("hess", False), w.get("sign") is not None), local)
    t_plan = time.perf_counter() - t_plan
    info = plan.info()
    B = len(w["nodes"])
    N = grid.num_nodes
    nodes_h = np.concatenate(w["nodes"]).astype(np.int64)
    offs_h = np.cumsum([0] + [len(n) for n in w["nodes"]]).astype(np.int64) if B > 1 else None
    sn_h, sw_h = (w["sign"] if w.get("sign") is not None else (None, None))

    def dev_t(x):
        return None if x is None else torch.from_numpy(np.ascontiguousarray(x)).to(dev)

    nodes_d, offs_d, sn_d, sw_d = dev_t(nodes_h), dev_t(offs_h), dev_t(sn_h), dev_t(sw_h)
    f64 = lambda: torch.empty(B * N, dtype=torch.float64, device=dev)  # noqa: E731
    outs = {"S": f64()}
    if w.get("grad"):
        outs["grad"] = [f64() for _ in range(dim)]
    if w.get("hess"):
        outs["hess"] = [f64() for _ in range(3)]
    if sn_d is not None:
        outs["mu"] = f64()
        outs["mask"] = torch.empty(B * N, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(profile=False):
        plan.run(nodes_d, offs_d, B, sn_d, sw_d, S=outs["S"], grad=outs.get("grad", (None,) * 3),
                 hess=outs.get("hess", (None,) * 3), mu=outs.get("mu"), mask=outs.get("mask"),
                 host=False, stream=stream.cuda_stream, profile=profile)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # per-pass device times (passes serialised, events between them), untimed
    pass_ms = {}
    for i in range(max(3, min(a.steps, 10))):
        flush.fill_(float(i))
        step(profile=True)
        for k, v in plan.pass_times().items():
            pass_ms.setdefault(k, []).append(v)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            flush.fill_(float(i))  # evict L2 between timed steps (outside the events)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            clk.sample()  # host-side, while the step runs on the device
        torch.cuda.synchronize()
    total_ms = reduce_max(dist, sum(s.elapsed_time(e) for s, e in ev), dev)
    if dist:
        dist.barrier()
    pts_per_step_job = B * N * world
    value = pts_per_step_job * a.steps / (total_ms / 1e3)

    # ---- phi validity band (untimed): fraction of nodes with phi >= 1e-5 / 1e-9 / 1e-13
    # (throughput counts every node, the valid band is reported beside it)
    phi_d = torch.empty(B * N, dtype=torch.float64, device=dev)
    plan.run(nodes_d, offs_d, B, None, None, phi=phi_d, host=False, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    validity = {f"phi>={t:g}": round(float((phi_d >= t).double().mean().item()), 6) for t in (1e-5, 1e-9, 1e-13)}
    del phi_d

    # ---- end to end through the C-ABI with pinned HOST buffers
    def pinned(n, dtype):
        return torch.empty(n, dtype=dtype, pin_memory=True).numpy()

    nodes_p = pinned(nodes_h.size, torch.int64)
    nodes_p[:] = nodes_h
    offs_p = None
    if offs_h is not None:
        offs_p = pinned(offs_h.size, torch.int64)
        offs_p[:] = offs_h
    sn_p = sw_p = None
    if sn_h is not None:
        sn_p = pinned(sn_h.size, torch.int64)
        sn_p[:] = sn_h
        sw_p = pinned(sw_h.size, torch.float64).reshape(sw_h.shape)
        sw_p[:] = sw_h
    ho = {"S": pinned(B * N, torch.float64)}
    d2h = B * N * 8
    if w.get("grad"):
        ho["grad"] = [pinned(B * N, torch.float64) for _ in range(dim)]
        d2h += dim * B * N * 8
    if w.get("hess"):
        ho["hess"] = [pinned(B * N, torch.float64) for _ in range(3)]
        d2h += 3 * B * N * 8
    if sn_h is not None:
        # the sign outputs: the winding number mu and the interior mask (classify's
        # rule with the flagged-node fill, R/sign.py:166-198)
        ho["mu"] = pinned(N, torch.float64)
        ho["mask"] = pinned(N, torch.uint8)
        d2h += 9 * N
    h2d = nodes_h.nbytes + (offs_h.nbytes if offs_h is not None else 16) + \
        ((sn_h.nbytes + sw_h.nbytes + 16) if sn_h is not None else 0)

    def e2e_step(wait=True):
        # wait=False: the call returns once queued (EIK_ASYNC); step i+1's column
        # passes overlap step i's device-to-host copies, and the last step waits
        plan.run(nodes_p, offs_p, B, sn_p, sw_p, S=ho["S"], grad=ho.get("grad", (None,) * 3),
                 hess=ho.get("hess", (None,) * 3), mu=ho.get("mu"), mask=ho.get("mask"),
                 host=True, stream=stream.cuda_stream, wait=wait)

    for _ in range(max(1, min(a.warmup, 3))):
        e2e_step()
    ke = max(3, min(a.steps, 10))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(ke):
        flush.fill_(1.0)
        e2e_step(wait=(i == ke - 1))
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = reduce_max(dist, e0.elapsed_time(e1), dev)
    e2e_val = pts_per_step_job * ke / (e2e_ms / 1e3)

    # ---- roofline of the dominant pass
    peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback"
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured"
    mean_pass = {k: float(np.mean(v)) for k, v in pass_ms.items()}
    alg = algorithmic_bytes(info, w, B)
    dom = max((k for k in mean_pass if k in alg), key=lambda k: mean_pass[k], default=None)
    roof = None
    if dom:
        # the dominant KERNEL's own duration (CUDA events around its launch inside the
        # pass); `pass_ms.col` also holds the small prep / row-DFT launches of the pass
        kern_ms = mean_pass.get("col_kernel") if dom == "col" and len(w["grid"].counts) == 2 else None
        ach = alg[dom] / ((kern_ms or mean_pass[dom]) / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(REPO, "profiles", "traffic.json")
        if os.path.exists(tpath):
            tj = json.load(open(tpath)).get(a.config, {})
            traffic = tj.get("col_kernel") if kern_ms and "col_kernel" in tj else tj.get(dom)
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": traffic, "kernel": "col_tmem_kernel (distance group)" if kern_ms else dom,
                "algorithmic_bytes": alg[dom],
                "kernel_ms": round(kern_ms or mean_pass[dom], 5), "pass_ms": round(mean_pass[dom], 5),
                "peak_source": peak_src,
                "peak_nominal": 8000.0, "frac_nominal": round(ach / 8000.0, 4),
                "step_bytes": sum(alg.values()),
                "step_frac": round(sum(alg.values()) / (total_ms / a.steps / 1e3) / 1e9 / peak, 4)}
        # SURVEY.md 8(d)'s looser "pruned, fused, out-of-core pass model" (B per
        # grid point: forward + inverse passes that each round-trip HBM), for
        # comparison with the survey's ideal Gpts/s; the tighter model above is
        # the one `frac` / `step_frac` use
        bpp = SURVEY_BYTES_PER_POINT.get(a.config)
        if bpp:
            sb = bpp * w["grid"].num_nodes * B
            roof["survey_pass_model"] = {"bytes_per_point": bpp, "step_bytes": sb,
                                         "step_frac": round(sb / (total_ms / a.steps / 1e3) / 1e9 / peak, 4)}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        wc = dict(w)
        if a.config == "C5":
            wc["nodes"] = w["nodes"][:8]
        v, sec, done, cores = cpu_time(wc, 1, 0)
        cpu = {"value": v, "unit": "grid_points/s", "cores": cores, "kind": "port",
               "sample": f"1 step of the oracle pipeline on {a.config}" + (" (8 items)" if a.config == "C5" else "")
                         + f" ({sec:.1f} s), scipy.fft workers={cores}"}

    # kernels per step (profiles/round2 launch lists): per group prep_nodes +
    # impulse_rows + column pass, then the row pass; C2 adds the sign mask fill
    # (flag bitmap + per-flagged-node search on a side stream + the gather behind the row
    # pass); 3-D adds the axis-1 lines passes
    launches_per_step = {"C1": 4, "C2": 10, "C3": 6, "C5": 4}[a.config]
    if rank == 0:
        line = {
            "metric": "grid points/sec (S+grad S+sign)", "value": value, "unit": "grid_points/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "strong" if a.config == "C5" else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators of BASELINE.json configs, workloads.py)",
            "config": {"workload": a.config, "desc": CONFIG_TEXT[a.config], "grid": list(grid.counts),
                       "batch_per_rank": B, "padded": list(info["padded"]), "l2": "flushed between timed steps",
                       "parallelism": parallelism(a.config, world, over),
                       "plan_build_s": round(t_plan, 3)},
            "e2e": {"value": e2e_val, "unit": "grid_points/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": ke,
                    "outputs": [k for k in ("S", "grad", "hess", "mu", "mask") if k in ho]},
            "gpu_launches": launches_per_step * a.steps,
            "pass_ms": {k: round(v, 5) for k, v in mean_pass.items()},
            "phi_validity": validity,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def bench_sweep(a):
    """tau sweep: 9 S fields from one transform of C2's delta_Y (single GPU / CPU oracle)."""
    from paper_1112_3010_b200 import workloads as wl

    d = wl.c2(a.seed)
    grid = d["grid"]
    nodes = d["points"].distinct_nodes()
    taus = [0.5 * (i + 1) for i in range(9)]
    pts = grid.num_nodes * len(taus)
    if a.impl == "reference":
        if int(os.environ.get("RANK", 0)) != 0:
            return 0
        import scipy.fft as sfft

        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import eikfld_oracle as orc

        cores = os.cpu_count() or 1
        with sfft.set_workers(cores):
            t0 = time.perf_counter()
            for tau in taus:  # the reference reuses the convolver but re-transforms per tau
                orc.phi_unchecked(nodes, grid.counts, 1.0, tau)
            sec = time.perf_counter() - t0
        v = pts / sec
        print(json.dumps({"metric": "grid points x taus/sec (tau sweep)", "value": v, "unit": "grid_points*taus/s",
                          "n_gpus": a.gpus, "steps": 1, "warmup": 0, "ms_per_step": sec * 1e3,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "impl": "reference", "config": {"workload": "TS", "taus": taus},
                          "cpu_baseline": {"value": v, "unit": "grid_points*taus/s", "cores": cores, "kind": "port",
                                           "sample": "one 9-tau sweep of the oracle"},
                          "e2e": {"value": v, "unit": "grid_points*taus/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return 0
    import torch

    from paper_1112_3010_b200 import _native

    dev = torch.device("cuda", 0)
    plan = _native.SweepPlan(2, grid.counts, grid.spacing, taus, 0)
    nd = torch.as_tensor(nodes, device=dev)
    outs = [torch.empty(grid.num_nodes, dtype=torch.float64, device=dev) for _ in taus]
    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        plan.run_sweep(nd, outs, host=False, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(stream)
        for _ in range(a.steps):
            plan.run_sweep(nd, outs, host=False, stream=stream.cuda_stream)
            clk.sample()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(json.dumps({"metric": "grid points x taus/sec (tau sweep)", "value": pts / (ms / 1e3),
                      "unit": "grid_points*taus/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
                      "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                      "dtype": "f64", "data": "synthetic", "config": {"workload": "TS", "taus": taus},
                      "gpu_launches": 6 * a.steps, "clocks": clk.summary()}))
    return 0


def bench_c4_single(a):
    """C4 on ONE GPU through eik_run: at 1024^3 the plan's fused buffers exceed the
    device, so the library runs its streamed schedule (one spectrum slot and one
    component slot live at a time, kernel spectra folded along all three axes);
    smaller --c4-size grids run the fused schedule."""
    import torch

    from paper_1112_3010_b200 import _native
    from paper_1112_3010_b200 import workloads as wl
    from paper_1112_3010_b200.engine import field_bits

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n = a.c4_size or 1024
    d = wl.c4(a.seed, n=n)
    grid = d["grid"]
    N = grid.num_nodes
    t_plan = time.perf_counter()
    plan = _native.Plan(3, grid.counts, grid.spacing, d["tau"], field_bits(3, True, False, True), 0)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t_plan
    nodes_h = np.ascontiguousarray(d["nodes"], dtype=np.int64)
    sn_h = np.ascontiguousarray(d["sign_nodes"], dtype=np.int64)
    sw_h = np.ascontiguousarray(d["sign_weights"], dtype=np.float64)
    nodes_d, sn_d, sw_d = (torch.as_tensor(x, device=dev) for x in (nodes_h, sn_h, sw_h))
    out = {"S": torch.empty(N, dtype=torch.float64, device=dev), "mu": torch.empty(N, dtype=torch.float64, device=dev),
           "mask": torch.empty(N, dtype=torch.uint8, device=dev),
           "grad": [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(3)]}

    def step(nd, sn, sw):
        plan.run(nd, None, 1, sn, sw, S=out["S"], grad=out["grad"], mu=out["mu"], mask=out["mask"], host=False)

    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        step(nodes_d, sn_d, sw_d)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    with ClockSampler(0) as clk:
        for i in range(a.steps):
            ev[i][0].record(stream)
            step(nodes_d, sn_d, sw_d)
            ev[i][1].record(stream)
            clk.sample()
        torch.cuda.synchronize()
    total_ms = sum(s_.elapsed_time(e_) for s_, e_ in ev)
    value = N * a.steps / (total_ms / 1e3)
    info = plan.info()
    free_b, tot_b = torch.cuda.mem_get_info(0)
    # size-independent check on the device (no oracle at this size): inside fraction of the
    # classified mask against the surface's enclosed volume, S >= 0 band near the surface
    inside = float(out["mask"].float().mean().item())
    # end to end: node lists from host memory, every field back to host memory
    e2e = None
    try:
        names = ["S", "mu", "mask", "g0", "g1", "g2"]
        srcs = [out["S"], out["mu"], out["mask"]] + out["grad"]
        host = {k: torch.empty(v.numel(), dtype=v.dtype, pin_memory=True) for k, v in zip(names, srcs)}
        d2h = sum(v.numel() * v.element_size() for v in host.values())
        h2d = nodes_h.nbytes + sn_h.nbytes + sw_h.nbytes
        ke = max(1, min(a.steps, 2))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            step(torch.as_tensor(nodes_h, device=dev), torch.as_tensor(sn_h, device=dev), torch.as_tensor(sw_h, device=dev))
            for k, v in zip(names, srcs):
                host[k].copy_(v, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e = {"value": N * ke / (e0.elapsed_time(e1) / 1e3), "unit": "grid_points/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": ke}
    except RuntimeError as exc:  # pinned host allocation of the fields refused
        e2e = {"value": None, "unit": "grid_points/s", "error": str(exc).splitlines()[0][:200]}
    plan.run(nodes_d, None, 1, sn_d, sw_d, S=out["S"], grad=out["grad"], mu=out["mu"], mask=out["mask"], host=False,
             profile=True)  # untimed: per-pass device times
    torch.cuda.synchronize()
    pt = plan.pass_times()
    peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback"
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured"
    step_s = total_ms / a.steps / 1e3
    sb = c4_step_bytes(grid.counts, info["padded"])
    roof = {"bound": "hbm", "achieved": round(sb / step_s / 1e9, 1), "peak": peak, "unit": "GB/s",
            "frac": round(sb / step_s / 1e9 / peak, 4), "traffic": None,
            "kernel": "whole step (chain of axis passes; fused-schedule pass model)", "algorithmic_bytes": sb,
            "peak_source": peak_src,
            "survey_pass_model": {"bytes_per_point": SURVEY_BYTES_PER_POINT["C4"], "step_bytes": SURVEY_BYTES_PER_POINT["C4"] * N,
                                  "step_frac": round(SURVEY_BYTES_PER_POINT["C4"] * N / step_s / 1e9 / peak, 4)}}
    line = {
        "metric": "grid points/sec (S+grad S+sign)", "value": value, "unit": "grid_points/s", "n_gpus": 1,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded perturbed icosphere, workloads.c4)",
        "config": {"workload": "C4" if n == 1024 else f"C4@{n}^3", "desc": CONFIG_TEXT["C4"], "grid": list(grid.counts),
                   "padded": list(info["padded"]), "vertices": int(d["vertices"].shape[0]),
                   "nodes": int(d["nodes"].size), "parallelism": "1 GPU (eik_run; streamed schedule when the fused "
                   "buffers exceed the device)", "l2": "working set >> L2", "plan_build_s": round(t_plan, 3),
                   "plan_bytes": int(info["device_bytes"]), "device_free_bytes_after": int(free_b),
                   "device_total_bytes": int(tot_b), "inside_fraction": round(inside, 6)},
        "e2e": e2e,
        "gpu_launches": None,
        "roofline": roof,
        "pass_ms": pt,
        "cpu_baseline": {"value": None, "unit": "grid_points/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": "infeasible: the reference pads to 3072^3 (464 GB per complex array) and "
                                   "caps FFTs at 2^31 elements (R/convolution.py:180-184)"},
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    return 0


def bench_c4(a):
    """C4: slab-decomposed 3-D pipeline, one rank per GPU, NCCL all-to-all between passes."""
    import torch

    rank, world, local = rank_env()
    if world == 1 and a.exchange != "nccl" and not os.environ.get("EIK_C4_SLAB"):
        return bench_c4_single(a)
    dist, local, over = init_ranks(world, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1112_3010_b200 import workloads as wl
    from paper_1112_3010_b200.slab import (CudaSlabExecutor, connect_p2p, fill_masks_emulated, fill_rank,
                                           local_nodes, nccl_exchange, run_rank, run_rank_p2p, run_rank_streamed,
                                           stream_barrier)

    # one fixed problem (1024^3) at every rank count: on fewer than 4 ranks the
    # fused schedule's 9 spectrum / component slots per rank exceed 180 GB, so
    # those run the streamed slab schedule (one V pair, one W pair, NCCL all-to-all)
    n = a.c4_size or 1024
    streamed = (n >= 1024 and world < 4) or os.environ.get("EIK_C4_STREAMED") == "1"
    d = wl.c4(a.seed, n=n)
    grid = d["grid"]
    t_plan = time.perf_counter()
    p2p = a.exchange == "p2p" and not streamed
    ex = CudaSlabExecutor(grid, d["tau"], world, rank, grad=True, sign=True, device=local, p2p=p2p,
                          streamed=streamed)
    t_plan = time.perf_counter() - t_plan
    ln, _ = local_nodes(d["nodes"], ex.layout)
    lsn, lsw = local_nodes(d["sign_nodes"], ex.layout, d["sign_weights"])
    ln_d, lsn_d, lsw_d = (torch.as_tensor(x, device=dev) for x in (ln, lsn, lsw))
    if p2p:
        # exchanges fused into the passes (peer stores into the owners' arenas)
        if dist:
            connect_p2p(ex, dist)
            barrier = stream_barrier(dist, dev)
        else:
            ex.plan.slab_p2p_connect(peer_arenas=[ex.arena])
            barrier = lambda: None  # noqa: E731

        def run_p2p(ex_, _exchange, *args):
            return run_rank_p2p(ex_, barrier, *args)
        run_schedule = run_p2p
        exchange = None
    elif dist:
        run_schedule = run_rank_streamed if streamed else run_rank
        exchange = nccl_exchange(dist)
    else:
        run_schedule = run_rank_streamed if streamed else run_rank

        def exchange(send, recv):
            for s_, r_ in zip(send, recv):
                r_.copy_(s_)

    def step(*args):
        # the config's sign output is the classified mask: fill the flagged nodes
        # from the neighbours' halo planes (classify, R/sign.py:166-198)
        out_ = run_schedule(ex, exchange, *args)
        if dist:
            fill_rank(ex, out_, d["sign_nodes"], dist)
        else:
            fill_masks_emulated([ex], [out_], d["sign_nodes"])
        return out_
    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        step(ln_d, lsn_d, lsw_d)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            ev[i][0].record(stream)
            out = step(ln_d, lsn_d, lsw_d)
            ev[i][1].record(stream)
            clk.sample()
        torch.cuda.synchronize()
    total_ms = reduce_max(dist, sum(s_.elapsed_time(e_) for s_, e_ in ev), dev)
    value = grid.num_nodes * a.steps / (total_ms / 1e3)
    # end to end: local node lists from host, the rank's fields back to pinned host memory
    host = {k: torch.empty(v.numel(), dtype=v.dtype, pin_memory=True) for k, v in
            [("S", out["S"]), ("mu", out["mu"]), ("mask", out["mask"])] + [(f"g{i}", g) for i, g in enumerate(out["grad"])]}
    d2h = sum(v.numel() * v.element_size() for v in host.values())
    h2d = ln.nbytes + lsn.nbytes + lsw.nbytes
    ke = max(1, min(a.steps, 3))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ke):
        o = step(ln, lsn, lsw)
        for k, v in host.items():
            src = o[k] if k in o else o["grad"][int(k[1])]
            v.copy_(src, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = reduce_max(dist, e0.elapsed_time(e1), dev)
    if rank == 0:
        L = ex.layout
        line = {
            "metric": "grid points/sec (S+grad S+sign)", "value": value, "unit": "grid_points/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded perturbed icosphere, workloads.c4)",
            "config": {"workload": "C4" if n == 1024 else f"C4@{n}^3", "desc": CONFIG_TEXT["C4"], "grid": list(grid.counts),
                       "padded": list(L.padded), "vertices": int(d["vertices"].shape[0]),
                       "nodes": int(d["nodes"].size),
                       "parallelism": parallelism("C4", world, over) + (
                           " (exchange fused into the passes: NVLink peer stores, 2 stream barriers; mask halo "
                           "planes point-to-point)" if p2p else
                           " (streamed: one input / one component at a time, NCCL all-to-all)" if streamed else
                           " (NCCL all-to-all)"),
                       "exchange_bytes_per_step": int(9 * 16 * L.buf * world * (world - 1) / world) if world > 1 else 0,
                       "l2": "working set >> L2", "plan_build_s": round(t_plan, 3)},
            "e2e": {"value": grid.num_nodes * ke / (e2e_ms / 1e3), "unit": "grid_points/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": ke},
            "gpu_launches": 12 * a.steps,
            "roofline": None,
            "cpu_baseline": {"value": None, "unit": "grid_points/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": "infeasible: the reference pads to 3072^3 (464 GB per complex array) and "
                                       "caps FFTs at 2^31 elements (R/convolution.py:180-184)"},
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
