"""The drop-in claim, proven with the reference's OWN tests on the B200.

tests/ref_plugin.py swaps ``ciphermlp.ckks.backend.CkksBackend`` for the B200
backend (plugin.install) in a subprocess pytest over the unmodified
reference test modules (baseline/_ref/ref_tests, vendored from
/root/reference by tools/vendor_reference.py; the reference package itself is
imported from baseline/_ref).  SURVEY.md §7 step 6 / §8(c) pinning tests:

  * tests/test_ckks_backend.py (all: encoding, ops tolerances, rotation group
    law, level exhaustion, cross-level alignment, debug-bootstrap contract,
    ledger parity with the simulator, RBCT / RBKY round trips, security gate);
  * acceptance C7 (CKKS correctness over 200 op cases, N=2^13) and C8 (two
    full unchanged ``train_iteration`` calls at N=2^13 within 2^-15 of the
    simulator, precision drop with injected refresh error);
  * tests/test_serialize.py[ckks] (the RBOT model container round trip after
    two training iterations), and the ckks cases of test_training / test_cli.
"""

import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "ref_tests")

SUITE = [
    "test_ckks_backend.py",
    "test_acceptance.py::test_criterion_7_ckks_correctness",
    "test_acceptance.py::test_criterion_8_ckks_end_to_end_microrun",
    "test_serialize.py::test_model_container_roundtrip",
    "test_training.py::test_ckks_requires_insecure_ack",
    "test_cli.py::test_ckks_insecure_gate",
]


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
@pytest.mark.skipif(not os.path.isdir(TESTS),
                    reason="baseline/_ref not vendored (tools/vendor_reference.py)")
def test_reference_ckks_suite_on_b200(tmp_path):
    report = tmp_path / "report.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, REF])
    env["CKB_REF_PLUGIN_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_plugin", "-p", "no:cacheprovider",
           "-o", "addopts=", "--rootdir", REF] + [os.path.join(TESTS, t) for t in SUITE]
    r = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-6000:]
    print(tail)
    assert r.returncode == 0, tail
    rep = json.loads(report.read_text())
    # the reference's tests really ran on the B200 class, through the sm_100a library
    assert rep["still_installed"] and rep["b200_backends_built"] >= 8, rep
    assert rep["native_library"].endswith("libckks_b200.so"), rep
