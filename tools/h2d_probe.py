"""Pinned host->device copy time vs size (torch and raw cudaMemcpyAsync)."""
import time
import torch

dev = torch.device("cuda:0")
for mb in [1, 4, 16, 64, 256, 1024]:
    n = mb * (1 << 20) // 8
    h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.int64, device=dev)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{mb:5d} MB  best {1e3*ts[0]:.3f} ms  median {1e3*ts[2]:.3f} ms  -> {mb/1024/ts[0]:.1f} GB/s")
