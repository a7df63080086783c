"""One warm split-and-merge training (fp32) for ncu launch lists / captures.
Usage: python tools/profile_step.py [config] [steps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import benchdata  # noqa: E402
from paper_1403_4781_b200 import _engine as E  # noqa: E402
from paper_1403_4781_b200.trainer import split_merge_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = benchdata.CONFIGS[name]
Ydev = benchdata.make_training_data_device(name, 1234, "fp32")
cap = cfg["s_max"] if cfg["eps"] is not None else cfg["s1"]
eps = cfg["eps"] or 0.0
for _ in range(steps):
    r = split_merge_device(Ydev, cfg["L"], cfg["K1"], cap, eps, cfg["local_iters"], cfg["K"],
                           cfg["s2"], cfg["merge_iters"], 1234, prec="fp32")
torch.cuda.synchronize()
print("done", r.wall_s)
