"""Run the reference's own unit tests against the drop-in.

  python tools/ref_suite.py prepare   # HERE (the reference is readable here)
  python tools/ref_suite.py run       # on the GPU box (gpurun)

`prepare` copies the reference's test files for the hot path
(pkg/tests/{conftest,reference,test_sparse_coding,test_dictionary_update,
test_trainer}.py) into the git-ignored baseline/_ref/suite/ (it travels to
the GPU box with the snapshot; nothing is committed) and writes a
`sparsedict` alias package in baseline/_ref/shim/ that IS
paper_1403_4781_b200 (sys.modules alias), so the tests run unchanged on the
GPU path in its default exact (FP64) mode. `run` executes pytest there and
writes gpurun_out/ref_suite.log + ref_suite.xml.
"""
import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SRC = Path("/root/reference/pkg/tests")
DST = ROOT / "baseline" / "_ref" / "suite"
SHIM = ROOT / "baseline" / "_ref" / "shim" / "sparsedict"
FILES = ["conftest.py", "reference.py", "test_sparse_coding.py", "test_dictionary_update.py",
         "test_trainer.py"]

SHIM_INIT = '''"""Test-only alias: the reference's tests import `sparsedict`; this makes
that name the B200 drop-in (paper_1403_4781_b200), default exact mode."""
import sys

import paper_1403_4781_b200 as _impl

sys.modules[__name__] = _impl
'''


def prepare():
    DST.mkdir(parents=True, exist_ok=True)
    for f in FILES:
        shutil.copy2(SRC / f, DST / f)
    SHIM.mkdir(parents=True, exist_ok=True)
    (SHIM / "__init__.py").write_text(SHIM_INIT)
    print(f"prepared {len(FILES)} files in {DST}")


def run():
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(SHIM.parent), str(ROOT), str(DST)])
    env["SDB_NO_BUILD"] = "1"
    cmd = [sys.executable, "-m", "pytest", str(DST), "-q", "-p", "no:cacheprovider", "--rootdir", str(DST),
           "-o", "addopts=", f"--junitxml={out / 'ref_suite.xml'}"]
    with open(out / "ref_suite.log", "w") as fh:
        rc = subprocess.run(cmd, cwd=str(DST), env=env, stdout=fh, stderr=subprocess.STDOUT).returncode
    print("rc", rc)
    return rc


if __name__ == "__main__":
    sys.exit({"prepare": prepare, "run": run}[sys.argv[1]]())
