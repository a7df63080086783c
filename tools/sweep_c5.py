"""BASELINE config 5: OMP coding-only sweep on one B200.

(m, K) in {(64,256),(64,1024),(144,576),(256,1024)}, s in {4,8,16,32},
N = 1,000,000 sparse-model signals (sigma = 0.01, generated on the GPU).
Per point: signals coded/s of the FP32 kernels alone and of the certified
path (FP32 kernels + sdb_certify: the reference's FP64 codes), CUDA events,
median of 3 after warm-up; the dominant kernel's roofline fraction
(k_omp_tc: useful TF32 flops vs the measured TF32 peak; k_corr_tc2: 3xTF32
flops vs the TF32 peak; k_omp_fast: L2 bytes 4*K*s per signal of G rows vs
the measured L2 read bandwidth, and HBM bytes vs HBM); parity of the
certified codes on a 20,000-signal sample vs the CPU oracle.
Prints one JSON object (profiles/c5_sweep_r02.json)."""
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import benchdata  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import parity as PA  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
points = [(64, 256), (64, 1024), (144, 576), (256, 1024)]
sparsities = [4, 8, 16, 32]
pk = bench.measure_peaks()
out = {"N": N, "precision": "fp32 (certified)", "peaks": pk, "points": []}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    res = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1000)
    return statistics.median(ts), res


for (m, K) in points:
    D = benchdata.gen_dictionary(m, K, 11)
    D32 = D.astype(np.float32).astype(np.float64)
    D32 /= np.linalg.norm(D32, axis=0)
    D64 = E.dict_to_device(D32)
    DT, G = E.working_dict(D64, "fp32"), E.gram(D64, "fp32")
    off, mx = E.shard_offsets([N])
    for s in sparsities:
        Yd = benchdata.sparse_signals_device(D, N, s, 0.01, 100 + s)
        t_raw, _ = timed(lambda: E.code(Yd, off, mx, DT, G, s, 0.0, "fp32", want_rnorm=False))
        t_cert, codes = timed(lambda: E.code_single_dict(Yd, D64, s, 0.0, "fp32", want_rnorm=False))
        E.KTIMER = {}
        E.code(Yd, off, mx, DT, G, s, 0.0, "fp32", want_rnorm=False)
        torch.cuda.synchronize()
        kt, E.KTIMER = E.KTIMER, None
        pt = {"m": m, "K": K, "s": s, "signals_per_s_fp32_kernels": N / t_raw,
              "signals_per_s_certified": N / t_cert, "ms_fp32": 1000 * t_raw, "ms_certified": 1000 * t_cert,
              "fragile": int(codes.nfrag.item()) if codes.nfrag is not None else None}
        for name, evs in kt.items():
            ms = sum(a.elapsed_time(b) for a, b, _, _ in evs)
            byts = sum(x for _, _, x, _ in evs)
            fl = sum(f for _, _, _, f in evs)
            k = {"ms": ms, "GBps": byts / (ms / 1e3) / 1e9}
            if name == "omp_tc":
                k.update(useful_tf32_tflops=fl / (ms / 1e3) / 1e12,
                         tensor_frac=fl / (ms / 1e3) / 1e12 / pk["tf32_tflops"], hbm_frac=k["GBps"] / pk["hbm_gbs"])
            elif name == "correlate":
                k.update(tensor_frac=3 * fl / (ms / 1e3) / 1e12 / pk["tf32_tflops"], hbm_frac=k["GBps"] / pk["hbm_gbs"])
            elif name == "omp":
                l2 = 4.0 * K * s * N
                k.update(hbm_frac=k["GBps"] / pk["hbm_gbs"],
                         l2_GBps=l2 / (ms / 1e3) / 1e9, l2_frac=l2 / (ms / 1e3) / 1e9 / pk.get("l2_read_gbs", 1e9))
            pt[name] = k
        # parity of the certified codes on a sample
        pick = np.sort(np.random.default_rng(11 + s).choice(N, 20_000, replace=False))
        gidx, gval, gcnt = PA.gpu_codes_host(codes, pick)
        Ys = E.d2h(Yd[torch.from_numpy(pick).to(Yd.device)]).astype(np.float64).T
        ref = O.omp_raw(Ys, D32, s, 0.0, threads=O.host_cores())
        par = PA.compare_codes(Ys, D32, gidx, gval, gcnt, ref, max_log=5)
        pt.update(parity_same_support=par["same_support"], parity_rel_fro=par["rel_fro"],
                  parity_divergent=par["n_divergent"])
        out["points"].append(pt)
        print(json.dumps(pt), file=sys.stderr, flush=True)
        del Yd, codes
        torch.cuda.empty_cache()
print(json.dumps(out))
