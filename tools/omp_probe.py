"""Time the OMP kernel on C5-style data under the call variants."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402

m, K, s, N = 64, 256, 4, 1_000_000
if len(sys.argv) > 3:
    m, K, s = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(3)
D = benchdata.gen_dictionary(m, K, 11) if hasattr(benchdata, "gen_dictionary") else None
if D is None:
    D = rng.standard_normal((m, K)); D /= np.linalg.norm(D, axis=0)
Y = benchdata.sparse_signals(D, N, s, 0.01, 5) if hasattr(benchdata, "sparse_signals") else None
if Y is None:
    X = np.zeros((K, N)); 
    for i in range(N):
        X[rng.choice(K, s, replace=False), i] = rng.standard_normal(s)
    Y = D @ X + 0.01 * rng.standard_normal((m, N))
Ydev, _ = E.ingest_signals(Y.T, "fp32")
D64 = E.dict_to_device(D)
off, mx = E.shard_offsets([N])
DT, G = E.working_dict(D64, "fp32"), E.gram(D64, "fp32")
ysq = E.signal_sq(Ydev)
for name, kw in [("default", {}), ("ysq+no_rnorm", dict(ysq=ysq, want_rnorm=False))]:
    for eps in (0.0, 0.05):
        for _ in range(2):
            E.code(Ydev, off, mx, DT, G, s, eps, "fp32", **kw)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            c = E.code(Ydev, off, mx, DT, G, s, eps, "fp32", **kw)
        b.record(); torch.cuda.synchronize()
        print(f"{name:14s} eps={eps}: {a.elapsed_time(b)/5:.3f} ms (corr+omp), mean n {c.counts.float().mean().item():.2f}")
