"""The unchanged reference layer code on the B200 backend, whole step.

tools/c1_dropin.py builds BASELINE config 1 (16 -> 8 -> 2, batch 32, N=2^12)
with the reference package's own ``keygen`` / ``build_model`` /
``prepare_sample`` / ``nn.train_iteration`` (nn.py:344-404, imported from
baseline/_ref).  With ``plugin.install`` active every HE call of that code
lands on the B200 backend.

* Mode A (the reference prime layout, numpy samplers, numpy FFT encoder):
  every ciphertext the step computes — the four updated weights/velocities
  handed to the refresh, and the four refreshed outputs — is byte-identical
  (RBCT, ckks/backend.py:210-222) to the reference CkksBackend's run of the
  same step (tests/golden/c1_modeA_digests.json, made by
  tests/golden/make_c1_modeA.py with the real reference).
* Mode B (BASELINE primes 60 + 8x40 + 60, HW-64 secret, device encoder):
  the decrypted weights after the step are within 1e-3 of the reference's.
"""

import json
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, os.path.join(ROOT, "tools"))

needs = [pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device"),
         pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "ciphermlp")),
                            reason="baseline/_ref not vendored (tools/vendor_reference.py)")]


@pytest.fixture()
def installed():
    import c1_dropin as C

    C.import_reference()
    from paper_2506_19693_b200 import plugin

    olds = []

    def install(**opts):
        cls, old = plugin.install(**opts)
        olds.append(old)
        return cls

    yield install
    for old in reversed(olds):
        plugin.uninstall(old)


def _gold(golden_dir):
    with open(os.path.join(golden_dir, "c1_modeA_digests.json")) as fh:
        return json.load(fh), np.load(os.path.join(golden_dir, "c1_modeA_weights.npy"))


@needs[0]
@needs[1]
def test_c1_step_mode_a_byte_identical_to_reference(installed, golden_dir):
    import c1_dropin as C

    gold, gold_w = _gold(golden_dir)
    cls = installed(prime_layout="reference", sampler="numpy", encoder="numpy")
    cust, model, shape, x, onehot = C.build()
    assert isinstance(cust.backend, cls)
    seen = C.capture_refresh_inputs(cust)
    C.step(cust, model, shape, x, onehot)
    assert seen == gold["refresh_inputs_sha256"]
    outs = [C.sha(cust.backend.serialize_cipher(pm.payload)) for pm in C.outputs(model)]
    assert outs == gold["outputs_sha256"]
    assert np.array_equal(C.weights(model, cust), gold_w)


@needs[0]
@needs[1]
def test_c1_step_baseline_primes_within_1e3_of_reference(installed, golden_dir):
    import c1_dropin as C

    _, gold_w = _gold(golden_dir)
    installed(prime_layout="baseline", secret_hw=64)
    cust, model, shape, x, onehot = C.build()
    assert cust.backend.chain.layout == "baseline"
    C.step(cust, model, shape, x, onehot)
    w = C.weights(model, cust)
    assert float(np.max(np.abs(w - gold_w))) <= 1e-3
