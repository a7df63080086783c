"""Where does an FP32 GPU training trajectory leave the FP64 oracle's?

For one shard of a BASELINE config, runs the alternating iteration on the
GPU (E.code -> E.mod_update -> E.replace_degenerate, exactly trainer._iteration)
and, from the SAME dictionary each iteration ("lockstep"), the oracle's
omp_codes -> mod_update -> replace_degenerate_atoms. Reports per iteration:
codes parity (supports, near-tie gaps), MOD output difference, unused /
replaced atom sets and replacement picks on both sides, and the drift of the
free-running trajectories.
usage: python tools/parity_trace.py c4 10 [c2 9 ...]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import benchdata  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import parity as PA  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.trainer import coding_mode, init_dictionaries  # noqa: E402

SEED = 1234


def shard_data(name, t):
    cfg = benchdata.CONFIGS[name]
    if cfg["kind"] == "sparse":
        Yd = benchdata.make_training_data_device(name, SEED)
    else:
        Yd = E.ingest_signals(benchdata.make_training_data(name, SEED).T, "fp32")[0]
    parts = O.split_indices(Yd.shape[0], cfg["L"], SEED)
    rows = torch.from_numpy(parts[t]).to(E.device())
    Ys = Yd.index_select(0, rows).contiguous()
    return cfg, Ys, O.derive_seeds(SEED, cfg["L"] + 1)[t]


def trace(name, t):
    cfg, Ys, seed = shard_data(name, t)
    n, m = Ys.shape
    S = E.ShardSet(Ys, E.shard_offsets([n])[0], [n], "fp32")
    cap, eps = coding_mode(m, cfg["K1"], cfg["s1"], cfg["eps"], cfg["s_max"])
    if cfg["eps"] is not None:
        cap = cfg["s_max"]
    Yh = E.d2h(Ys).astype(np.float64).T                       # m x n, the values the GPU trains on
    D = init_dictionaries(S, cfg["K1"], "first-columns", [seed])
    Dfree = O.init_dictionary(Yh, cfg["K1"], "first-columns", seed)
    print(json.dumps({"config": name, "shard": t, "n": n, "init_rel": float(
        np.linalg.norm(E.d2h(D[0]).T - Dfree) / np.linalg.norm(Dfree))}), flush=True)
    kw = dict(s=cap) if cfg["eps"] is None else dict(eps=eps, s_max=cap)
    for it in range(cfg["local_iters"]):
        Dh = E.d2h(D[0]).T.copy()                              # m x K f64 (this iteration's input)
        codes = E.code(S.Y, S.off, S.max_rows, E.working_dict(D, "fp32"), E.gram(D, "fp32"), cap, eps,
                       "fp32", True, ysq=S.signal_sq(), want_rnorm=False)
        r = E.mod_update(S, codes, D)
        Dmod = E.d2h(r.D[0]).T.copy()
        flags, nt = E.replace_degenerate(S, codes, r.D, r.usage)
        Dnew = E.d2h(r.D[0]).T.copy()
        fl = E.d2h(flags[0])
        # oracle from the same input dictionary
        X, _ = O.omp_codes(Yh, Dh, threads=16, **kw)
        gidx, gval, gcnt = PA.gpu_codes_host(codes)
        ref = O.omp_raw(Yh, Dh, cap, eps if cfg["eps"] is not None else 0.0, threads=16)
        par = PA.compare_codes(Yh, Dh, gidx, gval, gcnt, ref, eps=eps, max_log=10)
        Dm, resid, unused, rank, _ = O.mod_update(Yh, X, Dh)
        Dr, rep, unrep = O.replace_degenerate_atoms(Dm, Yh, X)
        g_unused = [int(a) for a in np.flatnonzero(E.d2h(r.dead[0]))]
        rec = {
            "it": it, "codes_same_support": par["same_support"], "codes_n_div": par["n_divergent"],
            "codes_rel_fro_same": par["rel_fro_same_support"], "max_gap": par["max_selection_gap"],
            "ties": [{k: v for k, v in x.items() if k in ("kind", "step", "gap", "eps_margin", "signal")}
                     for x in par["near_ties"][:5]],
            "mod_rel": float(np.linalg.norm(Dmod - Dm) / np.linalg.norm(Dm)),
            "unused_gpu": g_unused, "unused_ref": list(unused), "rank_gpu": int(r.rank[0].item()),
            "rank_ref": rank, "replaced_gpu": [int(a) for a in np.flatnonzero(fl == 1)],
            "replaced_ref": rep, "after_replace_rel": float(np.linalg.norm(Dnew - Dr) / np.linalg.norm(Dr)),
        }
        # free-running oracle trajectory
        Xf, _ = O.omp_codes(Yh, Dfree, threads=16, **kw)
        Dfm, *_ = O.mod_update(Yh, Xf, Dfree)
        Dfree, *_ = O.replace_degenerate_atoms(Dfm, Yh, Xf)
        rec["free_rel"] = float(np.linalg.norm(Dnew - Dfree) / np.linalg.norm(Dfree))
        if rep != rec["replaced_gpu"] or rec["after_replace_rel"] > 1e-4:
            # which data columns were picked for each target
            cols_ref = {a: int(np.argmax(np.abs(Yh.T @ Dr[:, a]))) for a in rep}
            cols_gpu = {a: int(np.argmax(np.abs(Yh.T @ Dnew[:, a]))) for a in rec["replaced_gpu"]}
            rec["picks_ref"], rec["picks_gpu"] = cols_ref, cols_gpu
            res_ref = np.linalg.norm(Yh - Dm @ O.csc_matrix(X), axis=0)
            top = np.argsort(-res_ref)[:6]
            rec["top_resid_ref"] = [(int(i), float(res_ref[i])) for i in top]
        print(json.dumps(rec), flush=True)
        D = r.D                                                # continue the GPU trajectory


if __name__ == "__main__":
    a = sys.argv[1:]
    for k in range(0, len(a), 2):
        trace(a[k], int(a[k + 1]))
