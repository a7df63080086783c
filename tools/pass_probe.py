"""One C2 local coding pass (2,040,200 permuted signals, 16 trained shard
dictionaries) through the fused (default) or the two-kernel (--plain) path.
Times it with CUDA events; the last repetition is bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off`."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.trainer import split_merge_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--plain", action="store_true")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

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
ysq = S.signal_sq()
DT, G = E.working_dict(Dl, "fp32"), E.gram(Dl, "fp32")
kw = dict(ysq=ysq, want_rnorm=args.plain)


def run():
    return E.code(Ys, off, mx, DT, G, cap, eps, "fp32", True, **kw)


for _ in range(2):
    c = run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(args.reps):
    c = run()
b.record()
torch.cuda.synchronize()
E.KTIMER = {}
for _ in range(args.reps):
    run()
torch.cuda.synchronize()
kt, E.KTIMER = E.KTIMER, None
per = {k: sum(x.elapsed_time(y) for x, y, _, _ in v) / len(v) for k, v in kt.items()}
print("per launch (ms): " + ", ".join(f"{k} {v:.3f}" for k, v in per.items()))
cnt = c.counts.cpu().numpy()
print(f"{'plain' if args.plain else 'fused'}: {a.elapsed_time(b) / args.reps:.3f} ms per pass; "
      f"mean n {cnt.mean():.3f}, n>=2 {(cnt >= 2).mean():.3f}, hist {np.bincount(cnt)[:6].tolist()}")
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
