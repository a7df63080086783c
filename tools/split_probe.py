import time, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1403_4781_b200 import _engine as E, _lib
import benchdata
N = 2040200
for rep in range(3):
    t0 = time.perf_counter(); a = _lib.permutation(N, 1234); t1 = time.perf_counter()
    b = np.random.default_rng(1234).permutation(N); t2 = time.perf_counter()
    p = E.split_permutation(N, 1234); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"native {1000*(t1-t0):.1f} ms  numpy {1000*(t2-t1):.1f} ms  native+pinned H2D {1000*(t3-t2):.1f} ms", flush=True)
import os; print("cores", len(os.sched_getaffinity(0)))
