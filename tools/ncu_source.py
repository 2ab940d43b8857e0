"""Per-source-line warp-stall samples from an ncu source-page CSV export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
res = []
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("",):
        try:
            samp = int(r[4] or 0)
        except ValueError:
            continue
        if samp > 0:
            d = dict(zip(hdr, r))
            top = sorted([(float(d[k] or 0), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k],
                         reverse=True)[:3]
            res.append((samp, cur, r[0], r[1][:100].strip(), top))
res.sort(reverse=True)
tot = sum(x[0] for x in res)
for x in res[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{x[0]:7d} {100 * x[0] / tot:5.1f}% {x[1]}:{x[2]:>4} {x[3][:80]:80s} {[(k, int(v)) for v, k in x[4]]}")
