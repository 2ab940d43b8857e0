"""Instruction mix of the hot kernels from `cuobjdump -sass` of the built library
(static SASS: proves the fp64 pipe mix, TMEM (STTM/LDTM), bulk-copy (UBLKCP)
and mbarrier (SYNCS) use, and the absence of local-memory traffic).

usage: python tools/sass_mix.py [lib.so] > profiles/round1/sass_mix.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1112_3010_b200/_lib/libeikfld_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
want = [("col_tmem_kernel<12, 1, 0, true>", r"col_tmem_kernelILi12ELi1ELi0ELb1E"),
        ("col_tmem_kernel<12, 1, 1, true>", r"col_tmem_kernelILi12ELi1ELi1ELb1E"),
        ("row_kernel<11, RCP>", r"row_kernelILi11ELb1EE"),
        ("impulse_rows_kernel<1, 8>", r"impulse_rows_kernelILi1ELi8EE"),
        ("col_tmem_kernel<9, 1, 0, true> (C3 axis 0)", r"col_tmem_kernelILi9ELi1ELi0ELb1E"),
        ("lines_kernel<9, true, false> (C3 axis 1 inverse)", r"lines_kernelILi9ELb1ELb0EE"),
        ("col_tmem_kernel<10, 1, 0, true> (C5)", r"col_tmem_kernelILi10ELi1ELi0ELb1E"),
        ("row_kernel<9> (C5)", r"row_kernelILi9ELb0EE")]
funcs = re.split(r"\n\s*Function : ", sass)
groups = {"fp64": ("DFMA", "DADD", "DMUL"), "tmem": ("STTM", "LDTM", "UTCATOMSWS", "UTCBAR"),
          "bulk/mbarrier": ("UBLKCP", "SYNCS"), "shared": ("LDS", "STS"), "global": ("LDG", "STG"),
          "local": ("LDL", "STL"), "barrier": ("BAR",), "prefetch": ("CCTL",)}
for label, pat in want:
    body = next((f for f in funcs if re.search(pat, f.split("\n", 1)[0])), None)
    if body is None:
        print(f"{label}: not found")
        continue
    ops = collections.Counter()
    for line in body.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            ops[m.group(2)] += 1
    tot = sum(ops.values())
    print(f"== {label}: {tot} static SASS instructions")
    for g, names in groups.items():
        c = {n: ops[n] for n in names if ops[n]}
        print(f"   {g:14s} {sum(c.values()):6d}  {c}")
