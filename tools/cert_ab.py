"""A/B check of two builds of the certification refit (sdb_certify): the same
seeded device data is coded by the FP32 kernels and certified by each library
(SDB_LIB=<path>, one subprocess per build); the certified FP64 coefficients,
supports and counts must be bitwise equal; each build's certify time is printed.
usage: cert_ab.py <lib_a.so> <lib_b.so>      (driver)
       cert_ab.py --run <out.npz>             (one build, via SDB_LIB)"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

# (P, n, K, s, m, eps)
SHAPES = [(256, 15625, 512, 8, 64, 0.0), (16, 127512, 256, 8, 64, 0.35), (32, 20000, 256, 5, 64, 0.0),
          (16, 7000, 200, 4, 36, 0.0), (1, 131072, 512, 4, 64, 0.0)]


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
        if eps > 0:   # mixed support sizes: some signals are (almost) one atom
            coef[:, 1:] *= (torch.rand(N, 1, device=dev, generator=g) > 0.5)
        shard = torch.arange(N, device=dev) // n
        Y = torch.einsum("ns,nsm->nm", coef, D[shard[:, None], sup])
        Y = (Y + 0.02 * torch.randn(N, m, device=dev, dtype=torch.float64, generator=g)).float().contiguous()
        del sup, coef
        off, mx = E.shard_offsets([n] * P)
        DT, G = E.working_dict(D, "fp32"), E.gram(D, "fp32")
        G64 = E.gram(D, "fp64")
        c = E.code(Y, off, mx, DT, G, s, eps, "fp32", want_rnorm=False, want_gap=True)

        def cert():
            return E.certify(Y, off, D, G64, E.DeviceCodes(c.K, c.cap, c.idx.clone(), c.val, c.counts.clone(),
                                                           c.status.clone(), c.rnorm, gap=c.gap), eps)
        for _ in range(2):
            cc = cert()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            cc = cert()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(f"  shape {k} P={P} n={n} K={K} s={s} m={m} eps={eps}: certify {ms:8.3f} ms, "
              f"fragile {int(cc.nfrag.item())}, mean support {cc.counts.float().mean().item():.2f}", flush=True)
        for f in ("idx", "val", "counts", "status"):
            res[f"{k}_{f}"] = getattr(cc, f).cpu().numpy()
    np.savez(out, **res)


def main():
    import numpy as np
    if sys.argv[1] == "--run":
        run(sys.argv[2])
        return
    outs = []
    for i, lib in enumerate(sys.argv[1:3]):
        out = f"/tmp/cert_ab_{i}.npz"
        print(f"build {i}: {lib}", flush=True)
        subprocess.run([sys.executable, __file__, "--run", out], check=True, env={**os.environ, "SDB_LIB": lib})
        outs.append(np.load(out))
    a, b = outs
    ok = True
    for key in a.files:
        if not np.array_equal(a[key], b[key], equal_nan=True):
            ok = False
            d = (a[key] != b[key])
            d = d.reshape(d.shape[0], -1).any(axis=1) if d.ndim > 1 else d
            rows = np.nonzero(d)[0][:6]
            print(f"DIFF {key}: {int(d.sum())} of {d.shape[0]} rows differ; rows {rows.tolist()}")
            print("   a", a[key][rows].reshape(len(rows), -1)[:, :8].tolist())
            print("   b", b[key][rows].reshape(len(rows), -1)[:, :8].tolist())
    print("bitwise equal" if ok else "NOT bitwise equal")


if __name__ == "__main__":
    main()
