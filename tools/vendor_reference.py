"""Install the UNMODIFIED reference package into baseline/_ref (git-ignored).

The GPU box has no /root/reference; baseline/_ref travels there with the repo
snapshot (git-ignored, not gpurun-ignored), so the drop-in tests
(tests/test_gpu_reference_suite.py: the reference's own CKKS tests with the
B200 backend installed through plugin.install) and bench.py's same-run CPU
reference legs (the reference CkksBackend timed on the box's host cores) can
import ``ciphermlp`` there.  Recipe (run by __graft_entry__.build() whenever
/root/reference is present):

  * ``pip install --no-index --no-build-isolation --no-deps --target
    baseline/_ref`` of a /tmp copy of /root/reference/pkg (the source tree is
    read-only and setuptools writes build files into it);
  * the reference's test modules copied to baseline/_ref/ref_tests so they run
    unchanged against the swapped class.

Nothing here is committed: baseline/_ref is listed in .gitignore.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = "/root/reference/pkg"
TARGET = os.path.join(ROOT, "baseline", "_ref")
STAMP = os.path.join(TARGET, ".vendored")


def _newest(path: str) -> float:
    t = 0.0
    for d, _, files in os.walk(path):
        for f in files:
            t = max(t, os.path.getmtime(os.path.join(d, f)))
    return t


def vendor(force: bool = False, verbose: bool = False) -> bool:
    """Returns True when baseline/_ref holds the reference package and tests."""
    if not os.path.isdir(REF_PKG):
        return os.path.exists(STAMP)
    if not force and os.path.exists(STAMP) and os.path.getmtime(STAMP) >= _newest(REF_PKG):
        return True
    shutil.rmtree(TARGET, ignore_errors=True)
    os.makedirs(TARGET)
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", TARGET, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{r.stdout[-2000:]}{r.stderr[-2000:]}")
    shutil.copytree(os.path.join(REF_PKG, "tests"), os.path.join(TARGET, "ref_tests"))
    with open(STAMP, "w") as fh:
        fh.write("pip install --target baseline/_ref /root/reference/pkg; tests -> ref_tests\n")
    if verbose:
        print(f"vendored the reference into {TARGET}")
    return True


if __name__ == "__main__":
    vendor(force="--force" in sys.argv, verbose=True)
