"""Time one FP32 coding pass at a C4-like shape (P shards x n signals, K atoms,
fixed sparsity s) through the fused tensor-core OMP (sdb_omp_tc) and the
two-launch path (tcgen05 GEMM + k_omp_fast). Data is generated on the device
with torch (timing probe only). Last repetition bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off`.
usage: omp_tc_probe.py [P n K s m]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1403_4781_b200 import _engine as E  # noqa: E402

P, n, K, s, m = 256, 15625, 512, 8, 64
if len(sys.argv) > 5:
    P, n, K, s, m = map(int, sys.argv[1:6])
only = sys.argv[6] if len(sys.argv) > 6 else None
dev = E.device()
g = torch.Generator(device=dev).manual_seed(1)
D = torch.randn(P, K, m, device=dev, dtype=torch.float64, generator=g)
D /= D.norm(dim=2, keepdim=True)
N = P * n
# s atoms per signal (uniform; a rare repeated atom is harmless for timing)
sup = torch.randint(0, K, (N, s), device=dev, generator=g)
coef = torch.randn(N, s, device=dev, dtype=torch.float64, generator=g)
shard = torch.arange(N, device=dev) // n
Y = torch.einsum("ns,nsm->nm", coef, D[shard[:, None], sup]) + 0.02 * torch.randn(N, m, device=dev, dtype=torch.float64, generator=g)
Y = Y.float().contiguous()
del sup, coef
torch.cuda.synchronize()
print(f"data ready: N={N} P={P} K={K} s={s} m={m}", flush=True)
off, mx = E.shard_offsets([n] * P)
DT, G = E.working_dict(D, "fp32"), E.gram(D, "fp32")
res = {}
for name, flag in (("omp_tc", True), ("two_launch", False)):
    if only and only != name:
        continue
    E.OMP_TC = flag
    for _ in range(2):
        c = E.code(Y, off, mx, DT, G, s, 0.0, "fp32", want_rnorm=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        c = E.code(Y, off, mx, DT, G, s, 0.0, "fp32", want_rnorm=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    res[name] = c
    print(f"{name:11s}: {ms:8.3f} ms per pass of {N} signals = {N / ms / 1e3:8.1f} M signals/s", flush=True)
if len(res) == 2:
    x, y = res["omp_tc"], res["two_launch"]
    si = torch.sort(x.idx, dim=1).values
    sj = torch.sort(y.idx, dim=1).values
    same = (si == sj).all(dim=1).float().mean().item()
    print(f"supports identical between the two paths: {same:.6f}; statuses equal "
          f"{(x.status == y.status).float().mean().item():.6f}")
E.OMP_TC = True
torch.cuda.profiler.start()
E.code(Y, off, mx, DT, G, s, 0.0, "fp32", want_rnorm=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
