"""standard (non-split) training on the whole dataset next to
split-and-merge, as a B200 number (the paper's comparison).

For a BASELINE config: train_standard semantics (one dictionary over all
signals, the config's K, coding mode and iteration count; trainer.py:165-197)
and the split-and-merge job, both device-resident in certified FP32; reports
wall time (CUDA events), OMP codings, final training MSE of each dictionary
coded over all signals (metrics.py:30-44) and, for the sparse-model configs,
atom recovery against the generating dictionary.
usage: python tools/standard_vs_split.py c4|c2 [precision]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.metrics import atom_recovery, mse_db_device  # noqa: E402
from paper_1403_4781_b200.trainer import (coding_mode, init_dictionaries, split_merge_device,  # noqa: E402
                                          train_device)

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
cfg = benchdata.CONFIGS[name]
SEED = 1234
Y = benchdata.make_training_data_device(name, SEED, prec)
N, m = Y.shape
cap, eps = coding_mode(m, cfg["K1"], cfg["s1"], cfg["eps"], cfg["s_max"])
if cfg["eps"] is not None:
    cap = cfg["s_max"]


def timed(fn):
    fn()                                   # warm-up (graph capture, workspaces)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1000.0, out


def quality(D64):
    S = E.ShardSet.single(Y, prec)
    c_final = cfg["s1"] * cfg["s2"] if cfg["eps"] is None else cap
    codes = E.code_single_dict(Y, D64, min(c_final, m), 0.0 if cfg["eps"] is None else eps, prec)
    q = {"final_mse_db": mse_db_device(S, codes, D64)}
    if cfg["kind"] == "sparse":
        q["atom_recovery_pct"] = atom_recovery(benchdata.gen_dictionary(m, cfg["K_true"], SEED), E.d2h(D64[0]).T)
    return q


def split():
    return split_merge_device(Y, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"], cfg["K"], cfg["s2"],
                              cfg["merge_iters"], SEED, prec=prec)


def standard():
    S = E.ShardSet.single(Y, prec)
    D0 = init_dictionaries(S, cfg["K"], "first-columns", [SEED])
    D, _, _ = train_device(S, D0, cap, eps, cfg["local_iters"])
    return D


t_split, r = timed(split)
t_std, Dstd = timed(standard)
out = {"config": name, "precision": prec, "N": N, "m": m, "K": cfg["K"], "iterations": cfg["local_iters"],
       "split_merge": {"train_s": t_split, "codings": r.codings, "codings_per_s": r.codings / t_split,
                       **quality(r.D_dev)},
       "standard": {"train_s": t_std, "codings": (cfg["local_iters"] + 1) * N,
                    "codings_per_s": (cfg["local_iters"] + 1) * N / t_std, **quality(Dstd)}}
print(json.dumps(out))
