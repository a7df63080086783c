"""Executed instructions and stall samples of one kernel by OUTERMOST source line
(the call site in the kernel body, following the inlined-at chains), grouped
into line ranges.
usage: ncu_regions.py <nvdisasm -gi output> <kernel substring> <ncu sass csv> <file.cu> lo-hi[:name] ...
  ncu -i X.ncu-rep --page source --csv --print-source sass > sass.csv
  cuobjdump -xelf all obj.o; nvdisasm -gi obj.sm_100a.cubin > dis.txt"""
import collections
import csv
import re
import sys

dis, kname, sass_csv, fname = sys.argv[1:5]
ranges = []
for s in sys.argv[5:]:
    rng, _, name = s.partition(":")
    lo, hi = rng.split("-")
    ranges.append((int(lo), int(hi), name or rng))

# offset -> outermost line in fname
outer = {}
infn = False
chain = []
for l in open(dis):
    s = l.strip()
    if s.startswith(".section") and ".text." in s:
        infn = kname in s
        continue
    if not infn:
        continue
    m = re.match(r'//## File ".*?/([^/"]+)", line (\d+)(?: inlined at ".*?/([^/"]+)", line (\d+))?', s)
    if m:
        chain.append(m)
        continue
    mo = re.match(r"/\*([0-9a-f]{4,6})\*/", s)
    if mo:
        if chain:
            last = chain[-1]
            if last.group(3):
                cur = (last.group(3), int(last.group(4)))
            else:
                cur = (last.group(1), int(last.group(2)))
            chain = []
        outer[int(mo.group(1), 16)] = cur

rows = list(csv.reader(open(sass_csv)))
h, data = rows[1], rows[2:]
ie, ns = h.index("Instructions Executed"), h.index("# Samples")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = [h.index(x) for x in reasons]
base = int(data[0][0], 16)
agg = collections.OrderedDict((r[2], [0.0, 0.0, collections.Counter()]) for r in ranges)
agg["other"] = [0.0, 0.0, collections.Counter()]
others = collections.Counter()
for r in data:
    off = int(r[0], 16) - base
    f, ln = outer.get(off, ("?", 0))
    key = "other"
    if f == fname:
        for lo, hi, name in ranges:
            if lo <= ln <= hi:
                key = name
                break
    a = agg[key]
    a[0] += float(r[ie] or 0)
    a[1] += float(r[ns] or 0)
    for x, i in zip(reasons, ri):
        a[2][x[6:]] += float(r[i] or 0)
    if key == "other":
        others[(f, ln)] += float(r[ns] or 0)
ti = sum(a[0] for a in agg.values())
ts = sum(a[1] for a in agg.values())
print(f"warp instructions {ti:.0f}, samples {ts:.0f}")
for k, a in agg.items():
    top = ", ".join(f"{n} {100 * c / max(a[1], 1):.0f}%" for n, c in a[2].most_common(4))
    print(f"{k:28s} instr {100 * a[0] / ti:5.1f}%  samples {100 * a[1] / ts:5.1f}%  [{top}]")
print("other (top):", others.most_common(6))
