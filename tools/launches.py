"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

UNIT = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}


def load(f):
    rows = list(csv.reader(open(f)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", "")) * UNIT[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += v
    return agg


if __name__ == "__main__":
    agg = load(sys.argv[1])
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
        print(f"{k:50s} {v[0]:5d} {v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}%")
    print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
