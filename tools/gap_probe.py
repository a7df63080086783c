"""GPU idle gaps inside one C2 split-and-merge job (torch profiler timeline)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.trainer import split_merge_device  # noqa: E402

cfg = benchdata.CONFIGS["c2"]
Yh = benchdata.make_training_data("c2")
Ydev, _ = E.ingest_signals(Yh.T, "fp32")
cap = cfg["s_max"] if cfg["eps"] is not None else cfg["s1"]


def job():
    return split_merge_device(Ydev, cfg["L"], cfg["K1"], cap, cfg["eps"] or 0.0, cfg["local_iters"], cfg["K"],
                              cfg["s2"], cfg["merge_iters"], 1234, prec="fp32")


for _ in range(3):
    job()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = job()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
busy, cur_s, cur_e = 0.0, None, None
gaps = []
for s, e, n in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            gaps.append((s - cur_e, cur_e, n))
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"span {(t1 - t0) / 1e3:.2f} ms, gpu busy {busy / 1e3:.2f} ms, idle {(t1 - t0 - busy) / 1e3:.2f} ms, "
      f"phases split {r.split_s*1e3:.2f} local {r.local_s*1e3:.2f} merge {r.merge_s*1e3:.2f}")
gaps.sort(reverse=True)
for g, at, n in gaps[:15]:
    print(f"  gap {g / 1e3:.3f} ms at +{(at - t0) / 1e3:.2f} ms before {n[:60]}")
