#!/usr/bin/env python
"""Benchmark: split-and-merge dictionary training on one B200 — OMP signals
coded per second over the whole training job (BASELINE.json metric "OMP
signals coded/sec and split-and-merge train time on 1 B200; % of roofline").

Default workload = the largest single-GPU configuration, C4 (BASELINE
configs[3]): N = 4,000,000 sparse-model signals (m=64, K_true=512, s=8,
sigma=0.02; generated on the GPU by sdb_synth_sparse), P=256 shards x local
K1=512 x 8 MOD iterations at fixed sparsity 8, then the merge K=512 from the
131,072 pooled scaled atoms (s2=4, 8 iterations; merge iterations are
unstated in BASELINE.json and chosen here). One step = one full split-and-
merge training on device-resident data; value = OMP signal-codings performed
in the job / job time (strong scaling: N GPUs share the shards, NCCL
all-gather of the local dictionaries, merge replicated). `--config c2`
selects BASELINE configs[1] (the error-bounded 8x8-patch job); the default
run also reports C2 under "extra".

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Under torchrun (N>1) every rank runs; rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import os

# the CPU leg must not oversubscribe: one BLAS thread per process
# (with default BLAS threads the process pool runs 4.6x slower)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import argparse  # noqa: E402
import ctypes  # noqa: E402
import gc  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import tempfile  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

UNIT = "signals/s"
CFG_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3}


def metric(cfg_name: str) -> str:
    return f"omp_signals_coded_per_s ({cfg_name.upper()} split-and-merge training job)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary C2 line")
    ap.add_argument("--groups", type=int, default=0,
                    help="concurrent shard groups in the local phase (device-resident run; 0: auto, "
                         "4 for >= 128 shards, else 1)")
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
def _peaks_lib():
    so = ROOT / "tools" / "_lat" / "libpeaks.so"
    if not so.exists():
        so.parent.mkdir(parents=True, exist_ok=True)
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-shared", "-Xcompiler", "-fPIC", "-o", str(so), str(ROOT / "tools" / "peaks.cu")],
                       check=True)
    lib = ctypes.CDLL(str(so))
    lib.peak_fma_f32.restype = ctypes.c_double
    lib.peak_l2_read.restype = ctypes.c_double
    lib.peak_l2_read.argtypes = [ctypes.c_int64]
    return lib


def measure_peaks() -> dict:
    """HBM and bf16 from the driver's MEASURED_PEAKS.json; TF32 (cuBLAS
    8192^3, allow_tf32), FP32 FFMA and L2 read bandwidth measured here, on
    this box, before the timed region (best of 3)."""
    import torch
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        hbm, bf16, src = float(d["hbm_gbs"]), float(d["bf16_tflops"]), "MEASURED_PEAKS.json (driver)"
    else:
        hbm, bf16, src = 6650.0, 1590.0, "fallback (B200_PROFILING.md)"
    out = {"hbm_gbs": hbm, "bf16_tflops": bf16, "hbm_bf16_source": src}
    try:
        old = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn(8192, 8192, device="cuda")
        b = torch.randn(8192, 8192, device="cuda")
        best = 0.0
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                torch.mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 5 * 2 * 8192 ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        torch.backends.cuda.matmul.allow_tf32 = old
        del a, b
        out["tf32_tflops"] = best
    except Exception as e:  # pragma: no cover
        out["tf32_tflops"] = bf16 / 2.0
        out["tf32_note"] = f"not measured ({e}); bf16/2"
    try:
        lib = _peaks_lib()
        out["fp32_simt_tflops"] = max(lib.peak_fma_f32() for _ in range(3))
        out["l2_read_gbs"] = max(lib.peak_l2_read(32 << 20) for _ in range(3))
    except Exception as e:  # pragma: no cover
        out["simt_l2_note"] = f"not measured ({e})"
    out["how"] = ("tf32: torch.mm 8192^3 fp32 with allow_tf32 (cuBLAS), best of 4x5; fp32_simt: 8 "
                  "independent FFMA chains/thread, 1184 CTAs x 256; l2_read: 32 MiB buffer swept 20x "
                  "with ld.global.cg float4 (tools/peaks.cu); best of 3")
    return out


def ncu_traffic() -> dict:
    """Per-launch DRAM bytes of the hot kernels from the committed ncu
    captures (profiles/ncu_*_raw.txt, one `ncu --set full` capture each)."""
    out = {}
    tags = (("k_omp_tc", "k_omp_tc"), ("k_omp_fast", None), ("k_corr_tc2", None))
    for f in sorted((ROOT / "profiles").glob("ncu_*_raw.txt")):
        vals = {}
        name = None
        for line in f.read_text().splitlines():
            parts = line.split()
            if line.startswith("Kernel Name"):
                name = None
                for base, fixed in tags:
                    if base + "<" in line:
                        if fixed:
                            name = fixed
                        else:
                            targs = line.split(base + "<", 1)[1].split(">", 1)[0].replace(" ", "").split(",")
                            flag = len(targs) >= 2 and targs[-1] in ("1", "true")
                            name = base + ("<DEFER>" if base == "k_omp_fast" and flag else
                                           "<CODE>" if flag else "")
            elif len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(parts[1], 1)
                vals[parts[0]] = float(parts[2]) * scale
            elif parts[:1] == ["capture:"]:
                vals["capture"] = " ".join(parts[1:])
        if name and "dram__bytes_read.sum" in vals and "dram__bytes_write.sum" in vals:
            out[name] = {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                         "file": f.name, "capture": vals.get("capture")}
    return out


# ----------------------------------------------------------------- CPU leg
def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_measure(cfg_name: str, Yh: np.ndarray, seed: int, cores: int, reps: int = 3,
                one_thread: bool = True) -> dict:
    """The oracle (reference algorithm: C OMP kernels restating _kernels.py +
    numpy/LAPACK MOD) on a bounded, representative sample of the job, then
    extrapolated to the whole job:

    * locals: 16 FULL-SIZE shards of the job's own split, ``its`` = 2 MOD
      iterations + the final coding pass each, one shard per worker process
      (1 BLAS thread each, like the reference's process pool,
      trainer.py:301-305) -> codings/s per shard-iteration on all cores; the
      same on one shard with one thread (1-core variant);
    * merge: one merge iteration on a pooled matrix of the job's full size
      (L x K1 scaled atoms; the sampled local dictionaries tiled to L) with
      all-core OMP -> seconds per merge pass;
    * job estimate = local codings / local rate + (merge_its + 1) merge passes.
    Repeated ``reps`` times: best and median reported; value = best."""
    import multiprocessing as mp

    import benchdata
    from oracle import oracle as O
    cfg = benchdata.CONFIGS[cfg_name]
    N, m = Yh.shape
    L, K1, its = cfg["L"], cfg["K1"], 2
    T = min(16, L)
    parts = O.split_indices(N, L, seed)[:T]
    seeds = O.derive_seeds(seed, L + 1)
    jobs = [(np.ascontiguousarray(Yh[p].T), K1, cfg["s1"], its, seeds[t], cfg["eps"], cfg["s_max"])
            for t, p in enumerate(parts)]
    n_sample = sum(len(p) for p in parts)
    cod_local = (its + 1) * n_sample
    t_all, t_one, locs = [], [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(min(cores, T)) as pool:
            locs = pool.map(O._local_job, jobs, chunksize=1)
        t_all.append(time.perf_counter() - t0)
    if one_thread:
        for _ in range(reps):
            t0 = time.perf_counter()
            O._local_job(jobs[0])
            t_one.append(time.perf_counter() - t0)
    # merge pass on the job-sized pooled matrix
    Ym = O.merge_dataset(locs)                                   # m x (T K1)
    Ym = np.tile(Ym, (1, L // T + 1))[:, :L * K1]
    n_merge = Ym.shape[1]
    t_merge = []
    for _ in range(max(1, reps - 1)):
        t0 = time.perf_counter()
        O.train_standard(Ym, cfg["K"], cfg["s2"], 1, "first-columns", seeds[L], threads=cores)
        t_merge.append((time.perf_counter() - t0) / 2.0)     # 2 coding passes + 1 MOD: per pass
    job_local = (cfg["local_iters"] + 1) * N
    job_codings = job_local + (cfg["merge_iters"] + 1) * n_merge
    rate_all_best = cod_local / min(t_all)
    rate_all_med = cod_local / statistics.median(t_all)
    tm = min(t_merge)
    job_s_best = job_local / rate_all_best + (cfg["merge_iters"] + 1) * tm
    job_s_med = job_local / rate_all_med + (cfg["merge_iters"] + 1) * statistics.median(t_merge)
    out = {
        "value": job_codings / job_s_best, "unit": UNIT, "cores": cores, "kind": "port",
        "median": job_codings / job_s_med, "job_s_est": job_s_best,
        "cpu_model": cpu_model(), "blas_threads_per_process": int(os.environ.get("OPENBLAS_NUM_THREADS", "0")),
        "locals_rate_all_cores": rate_all_best, "locals_s_per_shard_iteration_all_cores":
            min(t_all) / (T * (its + 1)) * min(cores, T),
        "merge_s_per_pass": tm,
        "sample": (f"oracle (C OMP restating _kernels.py + numpy/LAPACK MOD): {T} full-size shards "
                   f"({n_sample} signals) of the job's split x ({its} MOD iterations + final coding), "
                   f"one shard per process on {min(cores, T)} processes; 1 merge iteration on the "
                   f"{n_merge}-atom pooled matrix with {cores} OMP threads; extrapolated to the job "
                   f"({job_codings} codings); best of {reps} (median reported too)"),
    }
    if t_one:
        r1 = (its + 1) * len(parts[0]) / min(t_one)
        out["one_core"] = {"value": job_codings / (job_local / r1 + (cfg["merge_iters"] + 1) * tm * cores),
                           "locals_rate": r1, "cores": 1,
                           "note": "1 process, 1 BLAS thread; merge pass scaled by the core count"}
    return out


def reference_arm(args):
    """--impl reference: the reference algorithm on the host cores (the
    oracle port: the reference is Python/Numba and does not travel to the GPU
    box; the oracle's OMP is bitwise the reference's, its MOD the same LAPACK
    lstsq). Each step = the bounded, extrapolated sample of cpu_measure."""
    import benchdata
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    # host generator (same model; this arm touches no GPU code at all)
    Yh = benchdata.make_training_data(args.config, args.seed)
    cores = O.host_cores()
    for _ in range(args.warmup):
        cpu_measure(args.config, Yh, args.seed, cores, reps=1, one_thread=False)
    vals, secs, last = [], [], None
    for k in range(args.steps):
        last = cpu_measure(args.config, Yh, args.seed + k, cores, reps=1, one_thread=False)
        vals.append(last["value"])
        secs.append(last["job_s_est"])
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": metric(args.config), "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * float(np.median(secs)), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config.upper()} split-and-merge training (BASELINE "
                               f"configs[{CFG_INDEX[args.config]}]), extrapolated from a bounded sample",
                   "sample": last["sample"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": last["sample"], "cpu_model": last["cpu_model"]},
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


def time_steps(step, steps, world, clk=None):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # the interpreter's cyclic collector is paused over the timed region (a
    # generation-2 pass of the benchmark process stalls the launching thread
    # for tens of ms at a fixed call count); it runs right before instead
    gc.collect()
    gc_was = gc.isenabled()
    gc.disable()
    if clk:
        clk.mark(True)
    ev0.record()
    marks = []
    r = None
    for _ in range(steps):
        r = step()
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append(e)
    ev1.record()
    torch.cuda.synchronize()
    if gc_was:
        gc.enable()
    if clk:
        clk.mark(False)
    step_ms = [ev0.elapsed_time(marks[0])] + [a.elapsed_time(b) for a, b in zip(marks, marks[1:])]
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, step_ms, r


def make_step(cfg, Ydev, prec, seed, world, groups=1):
    from paper_1403_4781_b200.trainer import coding_mode, split_merge_device
    m = Ydev.shape[1]
    cap, eps = coding_mode(m, cfg["K1"], cfg["s1"], cfg["eps"], cfg["s_max"])
    if cfg["eps"] is not None:
        cap = cfg["s_max"]

    def step():
        if world > 1:
            from paper_1403_4781_b200.distributed import split_merge_ranks
            return split_merge_ranks(Ydev, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"],
                                     cfg["K"], cfg["s2"], cfg["merge_iters"], seed, prec=prec)
        return split_merge_device(Ydev, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"],
                                  cfg["K"], cfg["s2"], cfg["merge_iters"], seed, prec=prec, groups=groups)
    return step, cap


def kernel_breakdown(step, cfg, cap, m):
    """One eager step with CUDA events around every C-ABI call (on the
    launching stream); returns (breakdown, eager ms, deferred stats)."""
    import torch
    from paper_1403_4781_b200 import _engine as E
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
    kstat = dict(E.KSTAT)
    E.KSTAT.clear()
    deferred = int(kstat["deferred"].item()) if "deferred" in kstat else 0
    coded = int(kstat.get("coded", 0))
    K1 = cfg["K1"]
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
            breakdown[name]["flops_per_launch"] = fl / len(evs)
    if coded and "omp_deferred" in breakdown:
        breakdown["omp_deferred"]["deferred_fraction"] = deferred / coded
    return breakdown, ms_eager, omp_b


KERNEL_OF = {"omp": "k_omp_fast", "omp_deferred": "k_omp_fast<DEFER>", "correlate": "k_corr_tc2",
             "step1": "k_corr_tc2<CODE>", "omp_tc": "k_omp_tc"}


def roofline_of(name, d, pk, ms_eager, omp_b, m, K1, ncu):
    """Roofline object for one kernel of the breakdown. achieved = the
    kernel's ALGORITHMIC bytes or flops per launch / its average launch time
    (CUDA events on the launching stream, eager step)."""
    kname = KERNEL_OF[name]
    tr = ncu.get(kname)
    base = {"kernel": kname, "share_of_step": d["ms_per_step"] / ms_eager, "avg_launch_ms": d["avg_ms"],
            "traffic": tr["bytes"] if tr else None,
            "traffic_source": (f"ncu --set full, profiles/{tr['file']}" + (f" ({tr['capture']})" if tr.get("capture") else ""))
            if tr else None}
    if name == "omp_tc":
        ach = d["useful_TFLOPs"]
        t_tensor = d["flops_per_launch"] / (pk["tf32_tflops"] * 1e12)
        t_hbm = d["bytes_per_launch"] / (pk["hbm_gbs"] * 1e9)
        base.update(bound="tensor", achieved=ach, peak=pk["tf32_tflops"], unit="TFLOP/s",
                    frac=ach / pk["tf32_tflops"], peak_source="TF32 dense, measured on this box (cuBLAS)",
                    algorithmic="2*m*K TF32 flops per greedy step per signal (one D^T r MMA per step; "
                                "steps = atoms selected, i.e. s per signal at fixed sparsity)",
                    hbm_GBps=d["GBps"], hbm_frac=d["GBps"] / pk["hbm_gbs"],
                    bound_times_ms={"tensor": 1e3 * t_tensor, "hbm": 1e3 * t_hbm})
    elif name in ("omp", "omp_deferred"):
        base.update(bound="hbm", achieved=d["GBps"], peak=pk["hbm_gbs"], unit="GB/s",
                    frac=d["GBps"] / pk["hbm_gbs"], peak_source=pk["hbm_bf16_source"],
                    algorithmic_bytes_per_signal=omp_b + (8 if name == "omp_deferred" else 0))
    else:
        ach = 3 * d["useful_TFLOPs"]
        base.update(bound="tensor", achieved=ach, peak=pk["tf32_tflops"], unit="TFLOP/s",
                    frac=ach / pk["tf32_tflops"], peak_source="TF32 dense, measured on this box (cuBLAS)",
                    hbm_GBps=d["GBps"], hbm_frac=d["GBps"] / pk["hbm_gbs"],
                    algorithmic_flops_per_signal=3 * 2 * m * K1,
                    note="3xTF32 issues 3 MMAs per useful product (achieved counts all 3)")
    return base


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist

    import benchdata
    import paper_1403_4781_b200 as sdb

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = benchdata.CONFIGS[args.config]
    prec = args.precision
    pk = measure_peaks()
    Ydev = benchdata.make_training_data_device(args.config, args.seed, prec)   # resident in HBM
    N, m = Ydev.shape
    from paper_1403_4781_b200.trainer import auto_groups
    groups = args.groups or auto_groups(cfg["L"])
    step, cap = make_step(cfg, Ydev, prec, args.seed, world, groups)

    clk = Clocks(local)
    clk.ready()
    r = None
    for _ in range(args.warmup):
        r = step()
    codings = r.codings
    ms, step_ms, r = time_steps(step, args.steps, world, clk)
    print("per-step ms: " + " ".join(f"{x:.2f}" for x in step_ms), file=sys.stderr)
    clocks = clk.stop()
    value = codings / (ms / 1000.0)

    # per-kernel breakdown on one serial (single-group) eager step: concurrent
    # shard groups would overlap launches and blur per-launch durations
    step1, _ = make_step(cfg, Ydev, prec, args.seed, world, 1) if groups > 1 else (step, cap)
    breakdown, ms_eager, omp_b = kernel_breakdown(step1, cfg, cap, m)
    ncu = ncu_traffic()
    singles = {k: v for k, v in breakdown.items() if k in KERNEL_OF}
    dom = max(singles, key=lambda k: singles[k]["ms_per_step"]) if singles else None
    roof = roofline_of(dom, breakdown[dom], pk, ms_eager, omp_b, m, cfg["K1"], ncu) if dom else None
    others = {k: roofline_of(k, breakdown[k], pk, ms_eager, omp_b, m, cfg["K1"], ncu)
              for k in singles if k != dom}
    per_step = count_launches(step)
    gpu_launches = per_step * args.steps if per_step >= 0 else None

    # ---- e2e through the public API (sdb.train_split_merge) from host memory
    e2e = e2e_pageable = None
    Yh = None
    if not args.no_e2e or (rank == 0 and world == 1 and not args.no_cpu_baseline):
        Yh = Ydev.double().cpu().numpy()                    # (N, m) the values the device path trains on
    if not args.no_e2e:
        tc = sdb.TrainConfig(K=cfg["K"], s=cfg["s1"] * cfg["s2"], mode="split-merge",
                             L=cfg["L"], K1=cfg["K1"], s1=cfg["s1"], s2=cfg["s2"],
                             iterations=cfg["local_iters"], local_iterations=cfg["local_iters"],
                             merge_iterations=cfg["merge_iters"], seed=args.seed,
                             eps=cfg["eps"], s_max=cfg["s_max"], precision=prec)

        def e2e_run(Yin, reps):
            sdb.train_split_merge(Yin, tc, evaluate=False)
            torch.cuda.synchronize()
            gc.collect()
            gc_was = gc.isenabled()
            gc.disable()                 # as in time_steps
            t0 = time.perf_counter()
            for _ in range(reps):
                D, _ = sdb.train_split_merge(Yin, tc, evaluate=False)
            dt = (time.perf_counter() - t0) / reps
            if gc_was:
                gc.enable()
            return dt, D

        pinned = torch.empty((N, m), dtype=torch.float64, pin_memory=True)
        pinned.numpy()[:] = Yh
        t_e2e, D = e2e_run(pinned.numpy().T, max(1, args.steps))   # m x N view of pinned memory
        e2e = {"value": codings / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(N * m * 8),
               "d2h_bytes_per_step": int(D.nbytes), "ms_per_step": 1000 * t_e2e,
               "input": "pinned host f64 m x N (signal-major memory), train_split_merge(evaluate=False)"}
        del pinned
        Ypage = np.ascontiguousarray(Yh.T)                  # ordinary C-order m x N numpy array
        t_pg, D = e2e_run(Ypage, max(1, min(3, args.steps)))
        e2e_pageable = {"value": codings / t_pg, "unit": UNIT, "h2d_bytes_per_step": int(N * m * 8),
                        "d2h_bytes_per_step": int(D.nbytes), "ms_per_step": 1000 * t_pg,
                        "input": "pageable C-order m x N numpy f64 array, train_split_merge(evaluate=False)"}
        del Ypage

    # ---- secondary line: C2 (the error-bounded patch job), device-resident
    extra = None
    if args.config != "c2" and not args.no_extra and world == 1:
        c2 = benchdata.CONFIGS["c2"]
        Y2 = benchdata.make_training_data_device("c2", args.seed, prec)
        step2, cap2 = make_step(c2, Y2, prec, args.seed, 1)
        for _ in range(3):
            r2 = step2()
        ms2, _, r2 = time_steps(step2, 5, 1)
        bd2, eager2, ob2 = kernel_breakdown(step2, c2, cap2, Y2.shape[1])
        extra = {"c2": {"metric": metric("c2"), "value": r2.codings / (ms2 / 1000.0), "unit": UNIT,
                        "ms_per_step": ms2, "steps": 5, "warmup": 3,
                        "config": "BASELINE configs[1]: 2,040,200 DC-removed 8x8 patches, P=16, K1=K=256, "
                                  "eps=184, s<=16, 15 local + 15 merge iterations (s2=4)",
                        "kernels": bd2}}
        del Y2

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        cpu = cpu_measure(args.config, Yh, args.seed, O.host_cores())

    if rank == 0:
        line = {
            "metric": metric(args.config), "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic (sparse-model configs "
                                                                "generated on the GPU, sdb_synth_sparse)",
            "config": {"workload": f"{args.config.upper()} split-and-merge training (BASELINE "
                                   f"configs[{CFG_INDEX[args.config]}])",
                       "N": N, "m": m, "L": cfg["L"], "K1": cfg["K1"], "K": cfg["K"],
                       "local_iters": cfg["local_iters"], "merge_iters": cfg["merge_iters"],
                       "eps": cfg["eps"], "s_max": cfg["s_max"], "s1": cfg["s1"], "s2": cfg["s2"],
                       "codings_per_step": codings, "train_time_s": ms / 1000.0,
                       "phase_s": {"split": r.split_s, "locals": r.local_s, "merge": r.merge_s},
                       "precision": prec, "parallelism": f"shards over {world} GPU(s)", "shard_groups": groups,
                       "l2": "inputs larger than L2 (Y is %.0f MB)" % (N * m * 4 / 1e6)},
            "roofline": roof, "roofline_others": others, "peaks": pk, "kernels": breakdown,
            "kernels_note": f"per-kernel CUDA events from one extra eager single-group step ({ms_eager:.2f} ms; "
                            f"the timed steps replay CUDA graphs per training iteration, {groups} concurrent "
                            "shard group(s))",
            "cpu_baseline": cpu, "e2e": e2e, "e2e_pageable": e2e_pageable, "extra": extra,
            "gpu_launches": gpu_launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
