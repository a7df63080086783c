"""Phase times and GPU idle of train_split_merge on pinned host input (C2)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import benchdata  # noqa: E402
import paper_1403_4781_b200 as sdb  # noqa: E402

cfg = benchdata.CONFIGS["c2"]
Yh = benchdata.make_training_data("c2")
N, m = Yh.shape
pinned = torch.empty((N, m), dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = Yh
tc = sdb.TrainConfig(K=cfg["K"], s=cfg["s1"] * cfg["s2"], mode="split-merge", L=cfg["L"], K1=cfg["K1"],
                     s1=cfg["s1"], s2=cfg["s2"], iterations=cfg["local_iters"],
                     local_iterations=cfg["local_iters"], merge_iterations=cfg["merge_iters"], seed=1234,
                     eps=cfg["eps"], s_max=cfg["s_max"], precision="fp32")
for _ in range(3):
    D, rep = sdb.train_split_merge(pinned.numpy().T, tc, evaluate=False)
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    D, rep = sdb.train_split_merge(pinned.numpy().T, tc, evaluate=False)
    torch.cuda.synchronize()
    print(f"call {1e3*(time.perf_counter()-t):.2f} ms: split {1e3*rep.split_time_s:.2f} "
          f"locals {1e3*rep.local_wall_times_s[0]:.2f} merge {1e3*rep.merge_wall_time_s:.2f}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t = time.perf_counter()
    sdb.train_split_merge(pinned.numpy().T, tc, evaluate=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cs, ce = 0.0, None, None
for s, e in iv:
    if ce is None or s > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = s, e
    else:
        ce = max(ce, e)
busy += ce - cs
print(f"profiled wall {1e3*wall:.2f} ms; GPU span {(iv[-1][1]-iv[0][0])/1e3:.2f} ms, busy {busy/1e3:.2f} ms, "
      f"first kernel at +? ")
