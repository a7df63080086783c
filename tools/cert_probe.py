"""Certified FP32 coding cost at a C4-like shape: one coding pass over P
shards x n signals (device-generated sparse model, first-columns dictionary
per shard as in the first training iteration, then after two training
iterations), timing omp_tc, the FP64 refit and the exact re-run of the
fragile signals separately, and counting the fragile ones.
usage: cert_probe.py [P n K s m]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.trainer import _iteration, init_dictionaries  # noqa: E402

P, n, K, s, m = 256, 15625, 512, 8, 64
if len(sys.argv) > 5:
    P, n, K, s, m = map(int, sys.argv[1:6])
D_true = benchdata.gen_dictionary(m, K, 1234)
Y = E.synth_sparse(D_true, P * n, s, 0.02, 1235, "fp32")
S = E.ShardSet(Y, E.shard_offsets([n] * P)[0], [n] * P, "fp32")
D = init_dictionaries(S, K, "first-columns", list(range(P)))


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


for label in ("first-columns init", "after 2 iterations"):
    if label.startswith("after"):
        for _ in range(2):
            D, _ = _iteration(S, D, s, 0.0, True)
    DT, G = E.working_dict(D, "fp32"), E.gram(D, "fp32")
    G64 = E.gram(D, "fp64")
    t_tc, c = timed(lambda: E.code(S.Y, S.off, S.max_rows, DT, G, s, 0.0, "fp32", want_rnorm=False,
                                   want_gap=True))
    t_cert, cc = timed(lambda: E.certify(S.Y, S.off, D, G64, E.DeviceCodes(
        c.K, c.cap, c.idx.clone(), c.val, c.counts.clone(), c.status.clone(), c.rnorm, gap=c.gap), 0.0))
    nf = int(cc.nfrag.item())
    # refit only (no fragile signals): gap = +inf everywhere
    big = torch.full_like(c.gap, 1.0)
    t_refit, _ = timed(lambda: E.certify(S.Y, S.off, D, G64, E.DeviceCodes(
        c.K, c.cap, c.idx.clone(), c.val, c.counts.clone(), c.status.clone(), c.rnorm, gap=big), 0.0))
    t_g64, _ = timed(lambda: E.gram(D, "fp64"))
    gap = c.gap
    q = torch.quantile(gap[:1_000_000].float(), torch.tensor([1e-3, 1e-2, 0.1], device=gap.device))
    print(f"{label}: N={P * n} omp_tc {t_tc:.2f} ms | certify {t_cert:.2f} ms (refit only {t_refit:.2f} ms) "
          f"| gram64 {t_g64:.2f} ms | fragile {nf} ({100.0 * nf / (P * n):.3f}%) | gap quantiles "
          f"{[f'{x:.2e}' for x in q.tolist()]}", flush=True)
