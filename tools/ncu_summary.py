"""Summarise an ncu report: key metrics per kernel + top stall reasons."""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "--print-details", "all"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mi, vi, ii, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Stack Size", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "Local Memory Spilling Requests", "Shared Memory Configuration Size",
        "L1/TEX Cache Throughput", "Dynamic Shared Memory Per Block", "Block Limit Registers"]
seen = {}
for r in rows[1:]:
    if len(r) > vi and r[mi] in want:
        seen.setdefault((r[ii], r[ki][:60]), []).append(f"{r[mi]}={r[vi]}{r[ui]}")
for (i, k), v in seen.items():
    print(i, k)
    print("   " + "; ".join(v))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
for r in rr[2:]:
    if len(r) < len(h):
        continue
    name = r[h.index("Kernel Name")][:50]
    stalls = []
    for j, col in enumerate(h):
        m = re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_([a-z_]+)", col)
        if m and not m.group(1).endswith("not_issued"):
            try:
                stalls.append((float(r[j]), m.group(1)))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    stalls = [(100.0 * v / tot, n) for v, n in stalls]
    stalls.sort(reverse=True)
    extra = []
    for key in ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "smsp__inst_executed.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
                "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"):
        if key in h:
            extra.append(f"{key.split('.')[0]}={r[h.index(key)]}")
    print(name, "stall samples %:", ", ".join(f"{n}={v:.1f}" for v, n in stalls[:7]))
    print("   ", "; ".join(extra))
