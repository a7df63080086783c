"""Throughput of the zero-copy permuted gather from pinned host memory."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.trainer import split_merge_device  # noqa: E402

N, m = 2040200, 64
pinned = torch.empty((N, m), dtype=torch.float64, pin_memory=True)
import benchdata  # noqa: E402
pinned.numpy()[:] = benchdata.make_training_data("c2")
src = E.host_mapped(pinned.numpy())
perm = E.split_permutation(N, 1234)
bad = E.zeros((1,), torch.int32)
for rows in (N // 4, N):
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = E.ingest_gather(src, m, perm, 0, rows, m, "fp32", bad)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"gather {rows} rows from host: {1e3*dt:.2f} ms = {rows*m*8/dt/1e9:.1f} GB/s")
t = time.perf_counter()
d = pinned.to("cuda")
torch.cuda.synchronize()
print(f"plain H2D copy: {1e3*(time.perf_counter()-t):.2f} ms")
Ydev, _ = E.ingest_signals(pinned.numpy().T, "fp32")
for groups in (1, 2, 4):
    for _ in range(2):
        r = split_merge_device(Ydev, 16, 256, 16, 184.0, 15, 256, 4, 15, 1234, prec="fp32", groups=groups)
    print(f"device-resident groups={groups}: {1e3*r.wall_s:.2f} ms (split {1e3*r.split_s:.2f} locals {1e3*r.local_s:.2f} merge {1e3*r.merge_s:.2f})")
