"""A/B check of two builds of the fused tensor-core OMP (sdb_omp_tc): the same
seeded device data is coded by each library (SDB_LIB=<path>, one subprocess
per build); the outputs (idx, val, counts, status, gap) must be bitwise equal,
and each build's pass time is printed.
usage: omp_tc_ab.py <lib_a.so> <lib_b.so>      (driver)
       omp_tc_ab.py --run <out.npz>             (one build, via SDB_LIB)"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

# (P, n, K, s, m, eps)
SHAPES = [(256, 15625, 512, 8, 64, 0.0), (64, 8192, 512, 4, 64, 0.0), (32, 20000, 256, 5, 64, 0.0),
          (16, 7000, 200, 4, 36, 0.0), (32, 8000, 256, 8, 64, 0.3), (64, 15625, 512, 8, 64, 0.0),
          (16, 9000, 256, 5, 64, 0.0)]
FIRSTCOLS = {5, 6}


def run(out):
    import numpy as np
    import torch
    from paper_1403_4781_b200 import _engine as E
    dev = E.device()
    res = {}
    for k, (P, n, K, s, m, eps) in enumerate(SHAPES):
        g = torch.Generator(device=dev).manual_seed(11 + k)
        D = torch.randn(P, K, m, device=dev, dtype=torch.float64, generator=g)
        D /= D.norm(dim=2, keepdim=True)
        N = P * n
        sup = torch.randint(0, K, (N, s), device=dev, generator=g)
        coef = torch.randn(N, s, device=dev, dtype=torch.float64, generator=g)
        shard = torch.arange(N, device=dev) // n
        Y = torch.einsum("ns,nsm->nm", coef, D[shard[:, None], sup])
        Y = (Y + 0.02 * torch.randn(N, m, device=dev, dtype=torch.float64, generator=g)).float().contiguous()
        del sup, coef
        if k in FIRSTCOLS:   # first-columns initial dictionaries: the first K signals of a shard are its atoms
            D = Y.double().reshape(P, n, m)[:, :K, :].clone()
            D /= D.norm(dim=2, keepdim=True)
        off, mx = E.shard_offsets([n] * P)
        DT, G = E.working_dict(D, "fp32"), E.gram(D, "fp32")
        assert E.omp_tc_applies(m, K, s, "fp32")
        for _ in range(2):
            c = E.code(Y, off, mx, DT, G, s, eps, "fp32", want_rnorm=False, want_gap=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            c = E.code(Y, off, mx, DT, G, s, eps, "fp32", want_rnorm=False, want_gap=True)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(f"  shape {k} P={P} n={n} K={K} s={s} m={m} eps={eps}: {ms:8.3f} ms "
              f"({N / ms / 1e3:7.1f} M signals/s)", flush=True)
        for f in ("idx", "val", "counts", "status", "gap"):
            res[f"{k}_{f}"] = getattr(c, f).cpu().numpy()
    np.savez(out, **res)


def main():
    import numpy as np
    if sys.argv[1] == "--run":
        run(sys.argv[2])
        return
    outs = []
    for i, lib in enumerate(sys.argv[1:3]):
        out = f"/tmp/omp_tc_ab_{i}.npz"
        print(f"build {i}: {lib}", flush=True)
        subprocess.run([sys.executable, __file__, "--run", out], check=True, env={**os.environ, "SDB_LIB": lib})
        outs.append(np.load(out))
    a, b = outs
    ok = True
    for key in a.files:
        same = np.array_equal(a[key], b[key], equal_nan=True)
        if not same:
            ok = False
            d = (a[key] != b[key])
            d = d.reshape(d.shape[0], -1).any(axis=1) if d.ndim > 1 else d
            print(f"DIFF {key}: {int(d.sum())} of {d.shape[0]} rows differ")
            rows = np.nonzero(d)[0][:12]
            print("   rows", rows.tolist(), "a", a[key][rows].reshape(len(rows), -1)[:, :4].tolist(),
                  "b", b[key][rows].reshape(len(rows), -1)[:, :4].tolist())
    print("bitwise equal" if ok else "NOT bitwise equal")


if __name__ == "__main__":
    main()
