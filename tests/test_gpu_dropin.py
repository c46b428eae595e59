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


@needs[0]
@needs[1]
def test_c1_step_mode_a_deferred_byte_identical(installed, golden_dir):
    """deferred=True (deferred.py): the unchanged train_iteration's HE calls are
    recorded and run batched by the wave executor on the first decrypt /
    serialize — with the same bytes as the reference (and as eager)."""
    import c1_dropin as C

    gold, gold_w = _gold(golden_dir)
    installed(prime_layout="reference", sampler="numpy", encoder="numpy", deferred=True)
    cust, model, shape, x, onehot = C.build()
    seen = C.capture_refresh_inputs(cust)  # serializing the refresh inputs forces a flush
    C.step(cust, model, shape, x, onehot)
    outs = [C.sha(cust.backend.serialize_cipher(pm.payload)) for pm in C.outputs(model)]
    assert seen == gold["refresh_inputs_sha256"]
    assert outs == gold["outputs_sha256"]
    assert np.array_equal(C.weights(model, cust), gold_w)


@needs[0]
@needs[1]
def test_deferred_errors_surface_at_call_time(installed):
    """Deferred mode keeps the HE API's error timing: level exhaustion and
    missing keys from the base class, EncodingOverflow from the encode check."""
    import c1_dropin as C

    C.import_reference()
    from ciphermlp.api import keygen, make_plain
    from ciphermlp.errors import EncodingOverflow, LevelExhausted, MissingRotationKey
    from ciphermlp.params import make_params

    installed(deferred=True)
    params = make_params(level=2, scale_bits=40, poly_degree=2**10)
    cust = keygen(params, {1}, backend="ckks", rng_seed=1)
    slots = params.slot_count
    with pytest.raises(EncodingOverflow):
        cust.encrypt(make_plain(np.full(slots, 2.0**25), slots, 40.0))
    v = np.random.default_rng(0).uniform(-1, 1, slots)
    ct = cust.encrypt(make_plain(v, slots, 40.0))
    with pytest.raises(MissingRotationKey):
        cust.evaluator.rotate(ct, 2)
    x = ct
    for _ in range(2):
        x = cust.evaluator.mul(x, ct)
    with pytest.raises(LevelExhausted):
        cust.evaluator.mul(x, ct)
    got = cust.decrypt(cust.evaluator.rotate(ct, 1)).values
    assert np.max(np.abs(got - np.roll(v, -1))) < 1e-6


@needs[0]
@needs[1]
def test_c1_step_mode_a_pipelined_flush_byte_identical(installed, golden_dir):
    """deferred_async=True (pipelined flushes, deferred.py): the program is
    planned and issued on the worker thread while the caller goes on; the
    step's bytes equal the reference's, and two steps recorded back to back
    (step 2 reading step 1's pending outputs) equal a synchronous deferred run."""
    import c1_dropin as C

    gold, gold_w = _gold(golden_dir)
    installed(prime_layout="reference", sampler="numpy", encoder="numpy", deferred=True,
              deferred_async=True)
    cust, model, shape, x, onehot = C.build()
    seen = C.capture_refresh_inputs(cust)
    C.step(cust, model, shape, x, onehot)
    cust.backend.flush()  # returns at once
    outs = [C.sha(cust.backend.serialize_cipher(pm.payload)) for pm in C.outputs(model)]
    assert seen == gold["refresh_inputs_sha256"]
    assert outs == gold["outputs_sha256"]
    assert np.array_equal(C.weights(model, cust), gold_w)

    def two_steps(**opts):
        installed(prime_layout="reference", sampler="numpy", encoder="numpy", deferred=True,
                  **opts)
        cust, model, shape, x, onehot = C.build()
        for t in (1, 2):
            C.step(cust, model, shape, x, onehot, t=t)
            cust.backend.flush()
        return [C.sha(cust.backend.serialize_cipher(pm.payload)) for pm in C.outputs(model)]

    assert two_steps(deferred_async=True) == two_steps(deferred_async=False)
