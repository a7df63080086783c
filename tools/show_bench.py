"""Print the headline fields of a bench.py JSON line."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"ms/step {d['ms_per_step']:.2f}  value {d['value'] / 1e6:.1f}M/s  phases {d['config'].get('phase_s')}")
for k in ("roofline", "roofline_gemm"):
    r = d.get(k)
    if r:
        print(k, r["kernel"], f"{r['achieved']:.1f}/{r['peak']:.1f} {r['unit']} frac {r['frac']:.3f}",
              f"share {r.get('share_of_step', 0):.2f}")
for k, v in d.get("kernels", {}).items():
    print(f"  {k:14s} n={v['launches']:4d} {v['ms_per_step']:7.3f} ms/step avg {v['avg_ms']:.4f} ms "
          f"{v['GBps']:8.1f} GB/s" + (f" defer {v['deferred_fraction']:.3f}" if "deferred_fraction" in v else ""))
if d.get("e2e"):
    print("e2e", f"{d['e2e']['ms_per_step']:.2f} ms, {d['e2e']['value'] / 1e6:.1f}M/s")
