"""Time the pieces of the split phase of the C2 job on the device."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200 import trainer as T  # noqa: E402

cfg = benchdata.CONFIGS["c2"]
Yh = benchdata.make_training_data("c2")
Ydev, _ = E.ingest_signals(Yh.T, "fp32")
N = Ydev.shape[0]
L = cfg["L"]


def sync():
    torch.cuda.synchronize()


for rep in range(4):
    sync()
    t0 = time.perf_counter()
    perm = E.split_permutation(N, 1234)
    t1 = time.perf_counter()
    sync()
    t2 = time.perf_counter()
    Ys = E.gather_rows(Ydev, perm, "fp32")
    sync()
    t3 = time.perf_counter()
    base, extra = divmod(N, L)
    sizes = [base + (1 if t < extra else 0) for t in range(L)]
    off, _ = E.shard_offsets(sizes)
    S = E.ShardSet(Ys, off, sizes, "fp32")
    sync()
    t4 = time.perf_counter()
    seeds = T._derive_seeds(1234, L + 1)
    D0 = T.init_dictionaries(S, cfg["K1"], "first-columns", seeds[:L])
    sync()
    t5 = time.perf_counter()
    print(f"perm(host) {1e3*(t1-t0):.2f}  h2d {1e3*(t2-t1):.2f}  gather {1e3*(t3-t2):.2f}  "
          f"shards {1e3*(t4-t3):.2f}  init {1e3*(t5-t4):.2f} ms")
