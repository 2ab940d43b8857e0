"""Per-opcode / per-instruction stall summary from `ncu --page source --csv` (SASS view).

usage: ncu -i rep --page source --csv --print-kernel-base demangled > s.csv
       python tools/ncu_sass.py s.csv <kernel-substring> [ntop]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
want = sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 15
kern, hdr, ins = None, None, []
for r in rows:
    if r and r[0] == "Kernel Name":
        kern = r[1]
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if kern and want in kern and hdr and len(r) == len(hdr):
        ins.append(dict(zip(hdr, r)))
n = lambda i, k: int(i.get(k) or 0)
tot = sum(n(i, "# Samples") for i in ins) or 1
agg = {}
for i in ins:
    toks = i["Source"].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    a = agg.setdefault(op, [0, 0, 0, 0, 0])
    a[0] += n(i, "# Samples"); a[1] += n(i, "stall_long_sb"); a[2] += n(i, "stall_short_sb")
    a[3] += n(i, "stall_mio"); a[4] += n(i, "Instructions Executed")
print(f"{len(ins)} SASS instructions, {tot} samples")
for op, v in sorted(agg.items(), key=lambda x: -x[1][0])[:ntop]:
    print(f"{op:10s} samples {v[0]:7d} ({100 * v[0] / tot:4.1f}%) long_sb {v[1]:6d} short_sb {v[2]:6d} mio {v[3]:6d} exec {v[4]}")
loc = [i for i in ins if "LDL" in i["Source"] or "STL" in i["Source"]]
print("local-memory instructions:", len(loc), "executed", sum(n(i, "Instructions Executed") for i in loc))
top = sorted(range(len(ins)), key=lambda j: -n(ins[j], "# Samples"))[:ntop]
for j in top:
    print(f"{n(ins[j], '# Samples'):6d} lsb {n(ins[j], 'stall_long_sb'):5d} ssb {n(ins[j], 'stall_short_sb'):5d} "
          f"{ins[j]['Source'][:55]:55s} | prev: {ins[j - 1]['Source'][:45]}")
