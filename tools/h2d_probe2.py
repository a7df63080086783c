"""Where does the split permutation's host->device time go?"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1403_4781_b200 import _engine as E, _lib  # noqa: E402

N = 2040200
E.split_permutation(N, 1)
torch.cuda.synchronize()
host = E._pinned_perm[:N]
print("pinned:", host.is_pinned(), E._pinned_perm.is_pinned())
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.permutation(N, 1234, out=host.numpy())
    t1 = time.perf_counter()
    d = host.to(E.device(), non_blocking=True)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    d2 = host.to(E.device(), non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"perm {1e3*(t1-t0):.2f}  issue {1e3*(t2-t1):.3f}  copy {1e3*(t3-t2):.3f}  copy-again {1e3*(t4-t3):.3f} ms")
