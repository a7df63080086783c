"""How sensitive is the REFERENCE training itself to tiny input perturbations?

Trains one shard of a BASELINE config twice with the CPU oracle (FP64
restatement of the reference, trainer.py:165-197): once on Y, once on
Y * (1 + rel * xi), xi ~ N(0,1) per entry, and reports the relative Frobenius
distance of the two dictionaries after every iteration. If a 1e-12 input
perturbation already moves the reference's own dictionary by more than the
north_star's 1e-3 after the config's iteration count, no FP32 implementation
can meet that tolerance on that config (the training map amplifies near-tie
flips); parity must then be shown iteration by iteration (lockstep) and in the
GPU's FP64 mode.
usage: python tools/oracle_sensitivity.py c4 10 [rel ...]   (host data generator)"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import benchdata  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run(name, t, rels, seed=1234, threads=8):
    cfg = benchdata.CONFIGS[name]
    Y = benchdata.make_training_data(name, seed)
    Y = Y.astype(np.float32).astype(np.float64)
    part = O.split_indices(Y.shape[0], cfg["L"], seed)[t]
    Ys = np.ascontiguousarray(Y[part].T)
    s = O.derive_seeds(seed, cfg["L"] + 1)[t]
    kw = dict(s=cfg["s1"]) if cfg["eps"] is None else dict(eps=cfg["eps"], s_max=cfg["s_max"])
    rng = np.random.default_rng(7)
    xi = rng.standard_normal(Ys.shape)
    trajs = {}
    for rel in [0.0] + list(rels):
        Yp = Ys * (1.0 + rel * xi)
        D = O.init_dictionary(Yp, cfg["K1"], "first-columns", s)
        tr = []
        for it in range(cfg["local_iters"]):
            X, _ = O.omp_codes(Yp, D, threads=threads, **kw)
            D, *_ = O.mod_update(Yp, X, D)
            D, *_ = O.replace_degenerate_atoms(D, Yp, X)
            tr.append(D.copy())
        trajs[rel] = tr
    out = {"config": name, "shard": t, "n": Ys.shape[1], "iters": cfg["local_iters"], "rel_fro": {}}
    base = trajs[0.0]
    for rel in rels:
        out["rel_fro"][str(rel)] = [float(np.linalg.norm(a - b) / np.linalg.norm(b))
                                    for a, b in zip(trajs[rel], base)]
    return out


if __name__ == "__main__":
    name, t = sys.argv[1], int(sys.argv[2])
    rels = [float(x) for x in sys.argv[3:]] or [1e-12, 1e-9]
    print(json.dumps(run(name, t, rels)))
