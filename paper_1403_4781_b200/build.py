"""Build the sm_100a CUDA library in-tree: paper_1403_4781_b200/libsdb200.so.

    python -m paper_1403_4781_b200.build

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo; the .so travels to
the GPU box with the repo snapshot (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libsdb200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
OBJ = PKG / "build"


def sources():
    return sorted(CSRC.glob("*.cu"))


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(sources()) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + \
        [PKG.parent / "include" / "sparsedict_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    # one nvcc per translation unit in parallel, then one link
    OBJ.mkdir(exist_ok=True)
    jobs = []
    for src in sources():
        obj = OBJ / (src.stem + ".o")
        jobs.append((obj, [NVCC, *ARCH, *FLAGS, "-c", "-o", str(obj), str(src)]))
    if verbose:
        for _, cmd in jobs:
            print(" ".join(cmd), flush=True)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for r in ex.map(lambda j: subprocess.run(j[1]), jobs):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(LIB),
            *(str(o) for o, _ in jobs)]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
