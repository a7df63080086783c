"""Run a BASELINE config end to end on one B200 (device-resident split-and-
merge training, fp32 unless --fp64), report phase times, quality, and for C1
parity of the learned dictionary vs the CPU oracle on the same inputs.
Usage: python tools/run_config.py c1|c3|c4 [--fp64] [--no-oracle]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.metrics import mse_db_device  # noqa: E402
from paper_1403_4781_b200.trainer import coding_mode, split_merge_device  # noqa: E402

name = sys.argv[1]
prec = "fp64" if "--fp64" in sys.argv else "fp32"
cfg = benchdata.CONFIGS[name]
t0 = time.perf_counter()
Yh = benchdata.make_training_data(name, 1234)
gen_s = time.perf_counter() - t0
if prec == "fp32":
    Yh = Yh.astype(np.float32).astype(np.float64)
N, m = Yh.shape
Ydev, _ = E.ingest_signals(Yh.T, prec)
cap, eps = coding_mode(m, cfg["K1"], cfg["s1"], cfg["eps"], cfg["s_max"])
if cfg["eps"] is not None:
    cap = cfg["s_max"]
res = {}
for rep in range(2):  # first run warms up
    torch.cuda.synchronize()
    r = split_merge_device(Ydev, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"], cfg["K"],
                           cfg["s2"], cfg["merge_iters"], 1234, prec=prec)
res.update(config=name, precision=prec, N=N, m=m, L=cfg["L"], K1=cfg["K1"], K=cfg["K"],
           train_s=r.wall_s, split_s=r.split_s, locals_s=r.local_s, merge_s=r.merge_s,
           codings=r.codings, codings_per_s=r.codings / r.wall_s, datagen_s=gen_s,
           mem_peak_gb=torch.cuda.max_memory_allocated() / 1e9)
# quality: final coding of all data with the global dictionary (s = s1*s2 or eps)
S = E.ShardSet.single(Ydev, prec)
if cfg["eps"] is None:
    codes = E.code_single_dict(Ydev, r.D_dev, min(cfg["s1"] * cfg["s2"], m, cfg["K"]), 0.0, prec)
else:
    codes = E.code_single_dict(Ydev, r.D_dev, cfg["s_max"], cfg["eps"], prec)
res["final_mse_db"] = mse_db_device(S, codes, r.D_dev)
if name in ("c1", "c4"):
    Dt = benchdata.gen_dictionary(m, cfg["K_true"], 1234)
    from paper_1403_4781_b200.metrics import atom_recovery
    res["atom_recovery_pct"] = atom_recovery(Dt, r.D)
if name == "c1" and "--no-oracle" not in sys.argv:
    from oracle import oracle as O
    t1 = time.perf_counter()
    Dr, _ = O.split_merge(Yh.T, cfg["L"], cfg["K1"], cfg["s1"], cfg["local_iters"], cfg["K"],
                          cfg["s2"], cfg["merge_iters"], 1234, threads=8)
    res["oracle_s"] = time.perf_counter() - t1
    res["dict_rel_fro_vs_oracle"] = float(np.linalg.norm(r.D - Dr) / np.linalg.norm(Dr))
    res["dict_max_abs_vs_oracle"] = float(np.abs(r.D - Dr).max())
print(json.dumps(res))
