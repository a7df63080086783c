"""Timeline of train_split_merge on pinned host input (C2): per CUDA stream
span of its kernels, and when the host finished enqueuing each shard group."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import benchdata  # noqa: E402
import paper_1403_4781_b200 as sdb  # noqa: E402
from paper_1403_4781_b200 import trainer as T  # noqa: E402

cfg = benchdata.CONFIGS["c2"]
Yh = benchdata.make_training_data("c2")
N, m = Yh.shape
pinned = torch.empty((N, m), dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = Yh
tc = sdb.TrainConfig(K=cfg["K"], s=cfg["s1"] * cfg["s2"], mode="split-merge", L=cfg["L"], K1=cfg["K1"],
                     s1=cfg["s1"], s2=cfg["s2"], iterations=cfg["local_iters"],
                     local_iterations=cfg["local_iters"], merge_iterations=cfg["merge_iters"], seed=1234,
                     eps=cfg["eps"], s_max=cfg["s_max"], precision="fp32")
marks = []
_orig = T.train_device


def _wrapped(*a, **k):
    t = time.perf_counter()
    r = _orig(*a, **k)
    marks.append((t, time.perf_counter()))
    return r


T.train_device = _wrapped
for _ in range(3):
    D, rep = sdb.train_split_merge(pinned.numpy().T, tc, evaluate=False)
for _ in range(3):
    marks.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    D, rep = sdb.train_split_merge(pinned.numpy().T, tc, evaluate=False)
    torch.cuda.synchronize()
    print(f"call {1e3*(time.perf_counter()-t):.2f} ms: split {1e3*rep.split_time_s:.2f} "
          f"locals {1e3*rep.local_wall_times_s[0]:.2f} merge {1e3*rep.merge_wall_time_s:.2f}; "
          "host train_device spans (ms from call start): "
          + ", ".join(f"{1e3*(a-t):.1f}-{1e3*(b-t):.1f}" for a, b in marks))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sdb.train_split_merge(pinned.numpy().T, tc, evaluate=False)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
by = {}
for e in ev:
    s = by.setdefault(getattr(e, "device_resource_id", -1), [1e30, 0, 0, 0.0, {}])
    s[0] = min(s[0], e.time_range.start)
    s[1] = max(s[1], e.time_range.end)
    s[2] += 1
    s[3] += e.time_range.end - e.time_range.start
    nm = e.name.split("(")[0][:40]
    s[4][nm] = s[4].get(nm, 0.0) + e.time_range.end - e.time_range.start
for sid, (a, b, n, busy, names) in sorted(by.items(), key=lambda x: x[1][0]):
    top = sorted(names.items(), key=lambda x: -x[1])[:4]
    print(f"stream {sid}: {(a-t0)/1e3:7.2f} .. {(b-t0)/1e3:7.2f} ms, {n} kernels, busy {busy/1e3:.2f} ms; "
          + ", ".join(f"{k} {v/1e3:.2f}" for k, v in top))
