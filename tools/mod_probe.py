"""One C2 local MOD update (16 shards, K=256, m=64, codes of a trained
dictionary) timed with CUDA events; the last repetition is bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off`."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.trainer import split_merge_device  # noqa: E402

cfg = benchdata.CONFIGS["c2"]
Yh = benchdata.make_training_data("c2", 1234)
N, m = Yh.shape
Ydev, _ = E.ingest_signals(Yh.T, "fp32")
cap, eps = cfg["s_max"], cfg["eps"]
r = split_merge_device(Ydev, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"], cfg["K"], cfg["s2"],
                       cfg["merge_iters"], 1234, prec="fp32")
Dl = r.local_D
L = cfg["L"]
perm = E.split_permutation(N, 1234)
Ys = E.gather_rows(Ydev, perm, "fp32")
base, extra = divmod(N, L)
sizes = [base + (1 if t < extra else 0) for t in range(L)]
off, mx = E.shard_offsets(sizes)
S = E.ShardSet(Ys, off, sizes, "fp32")
codes = E.code(Ys, off, mx, E.working_dict(Dl, "fp32"), E.gram(Dl, "fp32"), cap, eps, "fp32", True,
               ysq=S.signal_sq(), want_rnorm=False)
u = E.code_usage(S, codes).cpu().numpy()
print(f"bucket sizes (entries per (shard, atom)): mean {u.mean():.0f} max {u.max()} p99 {np.percentile(u, 99):.0f} "
      f"top5 {np.sort(u.ravel())[-5:].tolist()}")
for _ in range(3):
    E.mod_update(S, codes, Dl)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    E.mod_update(S, codes, Dl)
b.record()
torch.cuda.synchronize()
print(f"mod_update: {a.elapsed_time(b) / 10:.3f} ms per call (16 shards)")
torch.cuda.profiler.start()
E.mod_update(S, codes, Dl)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
