#!/usr/bin/env python
"""Benchmark: split-and-merge dictionary training (BASELINE.json configs[1],
"C2") on B200 — OMP signals coded per second over the whole training job.

One step = one full split-and-merge training of C2 on device-resident data:
2,040,200 DC-removed 8x8 patches of 8 synthetic 512x512 images (sigma=20),
P=16 shards x local K1=256 x 15 MOD iterations with error-bounded OMP
(eps = 1.15*20*8 = 184, s <= 16), then the merge K=256 from the 4,096 pooled
scaled atoms (s2=4, 15 iterations; merge sparsity / iterations are unstated in
BASELINE.json and chosen here). value = OMP signal-codings performed in the
job / job time (strong scaling: N GPUs share the 16 shards, NCCL all-gather of
the local dictionaries, merge replicated).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Under torchrun (N>1) every rank runs; rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "omp_signals_coded_per_s (C2 split-and-merge training job)"
UNIT = "signals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--groups", type=int, default=1,
                    help="concurrent shard groups in the local phase (device-resident run)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1234)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampled every 200 ms during the timed region."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        self.t0 = self.t1 = None

    def ready(self, timeout: float = 5.0) -> None:
        """Block until the sampler has written its first line (its start-up
        NVML queries must not land inside the timed region)."""
        end = time.time() + timeout
        while self.p is not None and time.time() < end:
            if Path(self.f.name).stat().st_size > 0:
                return
            time.sleep(0.02)

    def mark(self, start: bool) -> None:
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        timed = []
        for r in rows:
            try:
                ts = time.mktime(time.strptime(r[0].strip().split(".")[0], "%Y/%m/%d %H:%M:%S")) + \
                    float("0." + r[0].strip().split(".")[1])
            except (ValueError, IndexError):
                ts = None
            if ts is not None and self.t0 is not None and self.t1 is not None and \
                    self.t0 - 0.05 <= ts <= self.t1 + 0.05:
                timed.append(r[1:])
        if timed:
            rows = timed
        else:
            rows = [r[1:] for r in rows]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for k, name in enumerate(names):
                if len(r) > 4 + k and r[4 + k].strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "window": "timed region" if timed else "whole sampler run"}


# ----------------------------------------------------------------- peaks
def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def ncu_traffic() -> dict:
    """Per-launch DRAM bytes of the hot kernels from the committed ncu captures."""
    out = {}
    for f in sorted((ROOT / "profiles").glob("ncu_*_raw.txt")):
        vals = {}
        name = None
        for line in f.read_text().splitlines():
            parts = line.split()
            if line.startswith("Kernel Name"):
                name = None
                for base, tag in (("k_omp_fast", "k_omp_fast<DEFER>"), ("k_corr_tc2", "k_corr_tc2<CODE>")):
                    if base + "<" in line:
                        targs = line.split(base + "<", 1)[1].split(">", 1)[0].replace(" ", "").split(",")
                        name = tag if len(targs) >= 2 and targs[-1] in ("1", "true") else base
            elif len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(parts[1], 1)
                vals[parts[0]] = float(parts[2]) * scale
        if name and len(vals) == 2:
            out[name] = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    return out


# ----------------------------------------------------------------- CPU sample
def cpu_sample(Yh: np.ndarray, cfg: dict, seed: int, threads: int):
    """The oracle (reference algorithm: C OMP kernels + numpy/LAPACK MOD) on a
    bounded sample of the same workload: 16 shards x 2,048 signals, 2 local
    and 2 merge iterations. Returns (codings/s, seconds, description)."""
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    L, K1 = cfg["L"], cfg["K1"]
    n = L * max(2048, K1)
    pick = np.sort(rng.choice(Yh.shape[0], size=min(n, Yh.shape[0]), replace=False))
    Ys = np.ascontiguousarray(Yh[pick]).T          # m x n (F-order view of signal-major rows)
    its = 2
    t0 = time.perf_counter()
    O.split_merge(Ys, L, K1, cfg["s1"], its, cfg["K"], cfg["s2"], its, seed,
                  eps=cfg["eps"], s_max=cfg["s_max"], threads=threads)
    dt = time.perf_counter() - t0
    codings = (its + 1) * Ys.shape[1] + (its + 1) * L * K1
    desc = (f"oracle split-merge on {Ys.shape[1]} of {Yh.shape[0]} signals: L={L}, K1={K1}, "
            f"{its} local + {its} merge iterations, same coding mode; {threads} OMP threads")
    return codings / dt, dt, desc


def reference_arm(args):
    """--impl reference: the reference algorithm on the host cores (oracle
    port: the reference's Python is not importable on the GPU box)."""
    import benchdata
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    cfg = benchdata.CONFIGS[args.config]
    Yh = benchdata.make_training_data(args.config, args.seed)
    cores = O.host_cores()
    for _ in range(args.warmup):
        cpu_sample(Yh, cfg, args.seed, cores)
    vals, secs = [], []
    for k in range(args.steps):
        v, dt, desc = cpu_sample(Yh, cfg, args.seed + k, cores)
        vals.append(v)
        secs.append(dt)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * float(np.mean(secs)), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config.upper()} split-and-merge training (bounded sample)",
                   "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def count_launches(step_fn) -> int:
    """Kernels of libsdb200 launched by one step (torch profiler / CUPTI)."""
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step_fn()
        n = 0
        for ev in prof.events():
            if ev.device_type.name == "CUDA" and "sdb::" in ev.name:
                n += 1
        return n
    except Exception:  # pragma: no cover - profiler unavailable
        return -1


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist

    import benchdata
    import paper_1403_4781_b200 as sdb
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200.trainer import split_merge_device, coding_mode

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = benchdata.CONFIGS[args.config]
    prec = args.precision
    Yh = benchdata.make_training_data(args.config, args.seed)       # (N, m) f64 host
    N, m = Yh.shape
    Ydev, bad = E.ingest_signals(Yh.T, prec)                         # resident in HBM
    cap, eps = coding_mode(m, cfg["K1"], cfg["s1"], cfg["eps"], cfg["s_max"])
    if cfg["eps"] is not None:
        cap = cfg["s_max"]

    def step():
        if world > 1:
            from paper_1403_4781_b200.distributed import split_merge_ranks
            return split_merge_ranks(Ydev, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"],
                                     cfg["K"], cfg["s2"], cfg["merge_iters"], args.seed,
                                     prec=prec)
        return split_merge_device(Ydev, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"],
                                  cfg["K"], cfg["s2"], cfg["merge_iters"], args.seed, prec=prec,
                                  groups=args.groups)

    clk = Clocks(local)
    clk.ready()
    for w in range(args.warmup):
        r = step()
    codings = r.codings
    # ---- timed region: barrier + sync on both sides, device-timed, max over ranks
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clk.mark(True)
    ev0.record()
    marks = []
    for _ in range(args.steps):
        r = step()
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append(e)
    ev1.record()
    torch.cuda.synchronize()
    clk.mark(False)
    step_ms = [ev0.elapsed_time(marks[0])] + [a.elapsed_time(b) for a, b in zip(marks, marks[1:])]
    print("per-step ms: " + " ".join(f"{x:.2f}" for x in step_ms), file=sys.stderr)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    # ---- per-kernel breakdown: one more step with CUDA events around every
    # C-ABI call (launched eagerly: events cannot sit inside a graph replay);
    # a first such step warms the event path up
    E.KTIMER = {}
    step()
    E.KTIMER = {}
    E.KSTAT.clear()
    E.KSTAT.update(deferred=E.zeros((1,), torch.int64), coded=0)
    torch.cuda.synchronize()
    eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eb0.record()
    step()
    eb1.record()
    torch.cuda.synchronize()
    ms_eager = eb0.elapsed_time(eb1)
    kt, E.KTIMER = E.KTIMER, None
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = codings / (ms / 1000.0)

    # ---- per-kernel breakdown (CUDA events recorded around each C-ABI call)
    hbm, bf16, peak_src = peaks()
    tf32_peak = bf16 / 2.0
    kstat = dict(E.KSTAT)
    E.KSTAT.clear()
    deferred = int(kstat["deferred"].item()) if "deferred" in kstat else 0
    coded = int(kstat.get("coded", 0))
    K1 = cfg["K1"]
    # algorithmic bytes per signal (fp32):
    #   omp (all signals): alpha0 row + ||y||^2 + code row (idx+val, cap wide) + count + status
    #   omp_deferred: the same per deferred signal + its (signal, shard) list entry
    #   step1: y row + ||y||^2 per signal; settled signals' code row + count + status;
    #          deferred signals' alpha0 row + list entry
    omp_b = 4 * K1 + 4 + 8 * cap + 5
    extra_bytes = {
        "omp_deferred": deferred * (omp_b + 8),
        "step1": (coded - deferred) * (8 * cap + 5) + deferred * (4 * K1 + 8),
    }
    breakdown = {}
    for name, evs in kt.items():
        tot = sum(a.elapsed_time(b) for a, b, _, _ in evs)
        byts = sum(x for _, _, x, _ in evs) + extra_bytes.get(name, 0)
        fl = sum(f for _, _, _, f in evs)
        breakdown[name] = {"launches": len(evs), "ms_per_step": tot,
                           "avg_ms": tot / len(evs), "GBps": byts / (tot / 1000.0) / 1e9,
                           "bytes_per_launch": byts / len(evs)}
        if fl > 0:
            breakdown[name]["useful_TFLOPs"] = fl / (tot / 1000.0) / 1e12
    if coded:
        breakdown["omp_deferred"]["deferred_fraction"] = deferred / coded
    # dominant single kernel (mod_update / replace are multi-kernel pipelines)
    kernel_of = {"omp": "k_omp_fast", "omp_deferred": "k_omp_fast<DEFER>",
                 "correlate": "k_corr_tc2", "step1": "k_corr_tc2<CODE>"}
    singles = {k: v for k, v in breakdown.items() if k in kernel_of}
    dom = max(singles, key=lambda k: singles[k]["ms_per_step"]) if singles else None
    roof = None
    ncu = ncu_traffic()
    if dom:
        d = breakdown[dom]
        kname = kernel_of[dom]
        if dom in ("omp", "omp_deferred"):
            roof = {"kernel": kname, "bound": "hbm", "achieved": d["GBps"], "peak": hbm, "unit": "GB/s",
                    "frac": d["GBps"] / hbm, "traffic": ncu.get(kname), "peak_source": peak_src,
                    "share_of_step": d["ms_per_step"] / ms_eager,
                    "algorithmic_bytes_per_signal": omp_b + (8 if dom == "omp_deferred" else 0)}
        else:
            ach = 3 * d["useful_TFLOPs"]
            roof = {"kernel": kname, "bound": "tensor", "achieved": ach, "peak": tf32_peak,
                    "unit": "TFLOP/s", "frac": ach / tf32_peak, "traffic": ncu.get(kname),
                    "peak_source": peak_src + "; TF32 dense = bf16/2",
                    "share_of_step": d["ms_per_step"] / ms_eager, "hbm_GBps": d["GBps"],
                    "hbm_frac": d["GBps"] / hbm,
                    "algorithmic_flops_per_signal": 3 * 2 * m * K1,
                    "note": "3xTF32 issues 3 MMAs per useful product (achieved counts all 3)"}
        roof["traffic_note"] = ("ncu dram read+write per launch of one C2 local pass (2,040,200 "
                                "signals), profiles/ncu_*_raw.txt")
    omp_roof = None
    oname = "omp_deferred" if "omp_deferred" in kt else ("omp" if "omp" in kt else None)
    if oname:
        d = breakdown[oname]
        omp_roof = {"kernel": kernel_of[oname], "bound": "hbm", "achieved": d["GBps"], "peak": hbm,
                    "unit": "GB/s", "frac": d["GBps"] / hbm, "traffic": ncu.get(kernel_of[oname]),
                    "share_of_step": d["ms_per_step"] / ms_eager,
                    "algorithmic_bytes_per_signal": omp_b + (8 if oname == "omp_deferred" else 0),
                    "note": "signals needing >= 2 atoms only (the fused GEMM epilogue settles the rest); "
                            "issue/latency bound, not HBM bound"}
    gemm = None
    gname = "step1" if "step1" in kt else ("correlate" if "correlate" in kt else None)
    if gname:
        d = breakdown[gname]
        gemm = {"kernel": kernel_of[gname], "bound": "tensor", "achieved": 3 * d["useful_TFLOPs"],
                "peak": tf32_peak, "unit": "TFLOP/s", "frac": 3 * d["useful_TFLOPs"] / tf32_peak,
                "useful_tflops": d["useful_TFLOPs"], "hbm_GBps": d["GBps"], "hbm_frac": d["GBps"] / hbm,
                "note": "3xTF32 issues 3 MMAs per useful product; TF32 dense peak = measured bf16/2"}
    # ---- launch count (one extra untimed step under the CUDA profiler)
    per_step = count_launches(step)
    gpu_launches = per_step * args.steps if per_step >= 0 else None

    # ---- e2e through the public API from pinned host memory (rank-local)
    e2e = None
    if not args.no_e2e:
        pinned = torch.empty((N, m), dtype=torch.float64, pin_memory=True)
        pinned.numpy()[:] = Yh
        Yview = pinned.numpy().T                  # m x N, F-order (no copy)
        tc = sdb.TrainConfig(K=cfg["K"], s=cfg["s1"] * cfg["s2"], mode="split-merge",
                             L=cfg["L"], K1=cfg["K1"], s1=cfg["s1"], s2=cfg["s2"],
                             iterations=cfg["local_iters"], local_iterations=cfg["local_iters"],
                             merge_iterations=cfg["merge_iters"], seed=args.seed,
                             eps=cfg["eps"], s_max=cfg["s_max"], precision=prec)
        sdb.train_split_merge(Yview, tc, evaluate=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(max(1, args.steps)):
            D, rep = sdb.train_split_merge(Yview, tc, evaluate=False)
        t_e2e = (time.perf_counter() - t0) / max(1, args.steps)
        e2e = {"value": codings / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(N * m * 8),
               "d2h_bytes_per_step": int(D.nbytes), "ms_per_step": 1000 * t_e2e}

    # ---- CPU baseline (rank 0, N=1 only, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        cores = O.host_cores()
        v, dt, desc = cpu_sample(Yh, cfg, args.seed, cores)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc,
               "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": f"{args.config.upper()} split-and-merge training (BASELINE "
                                   f"configs[{ {'c1': 0, 'c2': 1, 'c3': 2, 'c4': 3}[args.config]}])",
                       "N": N, "m": m, "L": cfg["L"], "K1": cfg["K1"], "K": cfg["K"],
                       "local_iters": cfg["local_iters"], "merge_iters": cfg["merge_iters"],
                       "eps": cfg["eps"], "s_max": cfg["s_max"], "s1": cfg["s1"], "s2": cfg["s2"],
                       "codings_per_step": codings, "train_time_s": ms / 1000.0,
                       "phase_s": {"split": r.split_s, "locals": r.local_s, "merge": r.merge_s},
                       "precision": prec, "parallelism": f"shards over {world} GPU(s)",
                       "l2": "inputs larger than L2 (Y is %.0f MB)" % (N * m * 4 / 1e6)},
            "roofline": roof, "roofline_gemm": gemm, "roofline_omp": omp_roof, "kernels": breakdown,
            "kernels_note": f"per-kernel events from one extra eager step ({ms_eager:.2f} ms; the timed "
                            "steps replay CUDA graphs per training iteration)", "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
