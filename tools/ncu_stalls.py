"""Stall reasons per SASS instruction from `ncu --page source --csv` output:
usage: ncu_stalls.py src.csv [addr_lo_suffix addr_hi_suffix] -- prints the
region's totals by reason and the top instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
src = h.index("Source")
ie = h.index("Instructions Executed")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = [h.index(x) for x in reasons]
sel = data
if len(sys.argv) > 3:
    a = [i for i, r in enumerate(data) if r[0].endswith(sys.argv[2])][0]
    b = [i for i, r in enumerate(data) if r[0].endswith(sys.argv[3])][0]
    sel = data[a:b + 1]
tot = {x: 0.0 for x in reasons}
for r in sel:
    for x, i in zip(reasons, ri):
        tot[x] += float(r[i] or 0)
s = sum(tot.values())
print(f"samples {s:.0f}: " + ", ".join(f"{k[6:]} {100 * v / s:.1f}%" for k, v in sorted(tot.items(), key=lambda t: -t[1]) if v > 0.005 * s))
top = sorted(sel, key=lambda r: -sum(float(r[i] or 0) for i in ri))[: int(sys.argv[4]) if len(sys.argv) > 4 else 25]
for r in top:
    v = {x: float(r[i] or 0) for x, i in zip(reasons, ri)}
    t = sum(v.values())
    main = ", ".join(f"{k[6:]} {c:.0f}" for k, c in sorted(v.items(), key=lambda t: -t[1])[:3] if c > 0)
    print(f"{r[0][-5:]} {t:6.0f} ex={r[ie]:>8s} {r[src][:70]:70s} [{main}]")
