"""BASELINE config 5: OMP coding-only sweep on one B200.

(m, K) in {(64,256),(64,1024),(144,576),(256,1024)}, s in {4,8,16,32},
N = 1,000,000 sparse-model signals (sigma = 0.01), FP32 fast mode.
Per point: signals coded/s (device-resident, CUDA events, median of 3 after
warm-up), the correlation GEMM's achieved TF32 tensor rate, the OMP kernel's
achieved HBM GB/s on its algorithmic bytes, and parity on a 2,000-signal
sample vs the CPU oracle (identical supports %, codes relative Frobenius).
Prints one JSON object; used for profiles/c5_sweep_r01.json.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import benchdata  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
points = [(64, 256), (64, 1024), (144, 576), (256, 1024)]
sparsities = [4, 8, 16, 32]
peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
out = {"N": N, "precision": "fp32", "points": []}
for (m, K) in points:
    D = benchdata.gen_dictionary(m, K, 11)
    D32 = D.astype(np.float32).astype(np.float64)
    D32 /= np.linalg.norm(D32, axis=0)
    for s in sparsities:
        Yh = benchdata.sparse_signals(D, N, s, 0.01, 100 + s)          # (N, m)
        Yd = torch.from_numpy(Yh.astype(np.float32)).cuda()
        D64 = E.dict_to_device(D32)
        DT, G = E.working_dict(D64, "fp32"), E.gram(D64, "fp32")
        off, mx = E.shard_offsets([N])
        for _ in range(2):
            E.code(Yd, off, mx, DT, G, s, 0.0, "fp32")
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            E.KTIMER = {}
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            codes = E.code(Yd, off, mx, DT, G, s, 0.0, "fp32")
            e1.record()
            torch.cuda.synchronize()
            kt = E.KTIMER
            E.KTIMER = None
            t = e0.elapsed_time(e1) / 1000
            corr_ms = sum(a.elapsed_time(b) for a, b, _, _ in kt["correlate"])
            omp_ms = sum(a.elapsed_time(b) for a, b, _, _ in kt["omp"])
            omp_bytes = sum(x for _, _, x, _ in kt["omp"])
            corr_flops = sum(f for _, _, _, f in kt["correlate"])
            times.append((t, corr_ms, omp_ms, omp_bytes, corr_flops))
        t, corr_ms, omp_ms, omp_bytes, corr_flops = sorted(times)[1]
        # parity on a sample
        ns = 2000
        Ys = Yh[:ns].astype(np.float32).astype(np.float64).T
        idx = E.d2h(codes.idx[:ns]); cnt = E.d2h(codes.counts[:ns]); val = E.d2h(codes.val[:ns])
        Xr, _ = O.omp_codes(Ys, D32, s=s, threads=8)
        ref = O.csc_matrix(Xr).toarray()
        got = np.zeros_like(ref)
        for i in range(ns):
            got[idx[i, :cnt[i]], i] = val[i, :cnt[i]]
        same = float(np.mean([np.array_equal(np.flatnonzero(ref[:, i]), np.flatnonzero(got[:, i])) for i in range(ns)]))
        rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        pt = {"m": m, "K": K, "s": s, "signals_per_s": N / t, "ms": 1000 * t,
              "corr_ms": corr_ms, "corr_tflops_3xtf32_useful": corr_flops / (corr_ms / 1000) / 1e12,
              "corr_frac_of_tf32_peak": corr_flops * 3 / (corr_ms / 1000) / 1e12 / (peaks["bf16_tflops"] / 2),
              "omp_ms": omp_ms, "omp_GBps": omp_bytes / (omp_ms / 1000) / 1e9,
              "omp_frac_hbm": omp_bytes / (omp_ms / 1000) / 1e9 / peaks["hbm_gbs"],
              "parity_same_support": same, "parity_rel_fro": rel}
        out["points"].append(pt)
        print(json.dumps(pt), file=sys.stderr, flush=True)
        del Yd, codes
        torch.cuda.empty_cache()
print(json.dumps(out))
