"""Per-source-line warp-stall samples and executed instructions from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` output.
usage: ncu_lines.py src.csv [min_pct]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) / 100 if len(sys.argv) > 2 else 0.004
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h, data = rows[hi], rows[hi + 1:]
ns, ie = h.index("# Samples"), h.index("Instructions Executed")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = [h.index(x) for x in reasons]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


per, cur, fname = collections.OrderedDict(), None, ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) < len(h) or r[0] == "Line No":
        continue
    if r[0] != "":
        cur = (fname, int(r[0]))
        per.setdefault(cur, [r[1], 0, 0, collections.Counter()])
        if r[2] == "":
            continue
    if r[2] != "" and cur is not None:
        per[cur][1] += f(r[ns])
        per[cur][2] += f(r[ie])
        for x, i in zip(reasons, ri):
            per[cur][3][x[6:]] += f(r[i])
tot = sum(v[1] for v in per.values())
tote = sum(v[2] for v in per.values())
print("total samples", tot, "warp instructions", tote)
for ln, v in sorted(per.items()):
    if v[1] > thr * tot or v[2] > thr * tote:
        top = ", ".join(f"{k} {c:.0f}" for k, c in v[3].most_common(3))
        print(f"{ln[0][:14]:14s}{ln[1]:4d} s={100 * v[1] / tot:5.1f}% i={100 * v[2] / tote:5.1f}% {v[0].strip()[:78]:78s} [{top}]")
