"""Config 1 through the UNCHANGED reference layer code (the real drop-in).

BASELINE config 1: MLP 16 -> 8 -> 2 with local-error-signal heads, batch 32,
x ~ U[-1,1]^16, one-hot labels from a seeded random linear teacher,
Xavier-uniform init, one encrypted forward + local backward + SGD step at
N=2^12, scale 2^40.  Everything here calls the
reference package ``ciphermlp`` (imported from baseline/_ref on the GPU box,
from /root/reference/pkg/src in the build container): ``keygen``,
``build_model``, ``encrypt_packed``, ``prepare_sample`` and
``nn.train_iteration`` (nn.py:344-404) run unmodified; with
``paper_2506_19693_b200.plugin.install`` active, ``backend="ckks"`` is the
B200 backend, otherwise it is the reference's numpy ``CkksBackend``.

Used by tests/golden/make_c1_modeA.py (reference digests), by
tests/test_gpu_dropin.py (mode-A whole-step bit identity on the B200) and by
bench.py (the c1 step timed through the layer code on the B200 next to the
reference CkksBackend on the same host).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIRS = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


def import_reference():
    """Make ``ciphermlp`` importable (vendored copy first); returns the package."""
    try:
        import ciphermlp  # noqa: F401
    except ImportError:
        for d in REF_DIRS:
            if os.path.isdir(os.path.join(d, "ciphermlp")):
                sys.path.insert(0, d)
                break
    import ciphermlp

    return ciphermlp


def setup(batch: int = 32):
    """Config-1 data and Xavier-uniform init (seeded)."""
    import_reference()
    from ciphermlp.packing import Architecture, compute_dims

    arch = Architecture(16, (8,), 2)
    n = 2**12
    rng = np.random.default_rng(20250624)
    x = rng.uniform(-1, 1, size=(32, 16))
    teacher = rng.normal(size=(16, 2))
    onehot = np.eye(2)[np.argmax(x @ teacher, axis=1)]
    w1 = rng.uniform(-1, 1, size=(16, 8)) * np.sqrt(6.0 / (16 + 8))
    c1 = rng.uniform(-1, 1, size=(8, 2)) * np.sqrt(6.0 / (8 + 2))
    shape = compute_dims(arch, n // 2)
    return arch, n, x[:batch], onehot[:batch], w1, c1, shape


def build(batch: int = 32, **keygen_opts):
    """keygen + build_model + Xavier weights re-encrypted (as the reference's
    tests do, tests/test_nn.py:125)."""
    from ciphermlp.api import keygen
    from ciphermlp.depth import tau_total
    from ciphermlp.nn import Hyperparams, build_model, classifier_format, layer_format
    from ciphermlp.packing import encrypt_packed, pack, required_rotations
    from ciphermlp.params import make_params

    arch, n, x, onehot, w1, c1, shape = setup(batch)
    params = make_params(level=tau_total(1), scale_bits=40, poly_degree=n)
    cust = keygen(params, required_rotations(shape), backend="ckks", rng_seed=3, **keygen_opts)
    hyper = Hyperparams(learning_rate=0.05, momentum=0.9, iterations=1, batch_size=batch,
                        rng_seed=0)
    model = build_model(arch, params, hyper, cust)
    blk = model.blocks[0]
    blk.layer_weights = encrypt_packed(cust, pack(w1, layer_format(blk.kind), shape))
    blk.classifier_weights = encrypt_packed(cust, pack(c1, classifier_format(blk.kind), shape))
    return cust, model, shape, x, onehot


def step(cust, model, shape, x, onehot, t: int = 1):
    """One config-1 step: encrypt the batch (prepare_sample) + train_iteration."""
    from ciphermlp.nn import prepare_sample, train_iteration

    batch = [prepare_sample(x[i], onehot[i], shape, cust) for i in range(x.shape[0])]
    train_iteration(model, batch, cust, t)
    return model


def outputs(model):
    b = model.blocks[0]
    return [b.layer_weights, b.classifier_weights, b.layer_velocity, b.classifier_velocity]


def sha(blob: bytes) -> str:
    return hashlib.sha256(blob).hexdigest()


def capture_refresh_inputs(cust):
    """Record the RBCT digest of every ciphertext handed to the refresh (the
    updated weights and velocities before the debug bootstrap)."""
    be = cust.backend
    seen = []
    orig = be.bootstrap

    def bootstrap(cv):
        seen.append(sha(be.serialize_cipher(cv)))
        return orig(cv)

    be.bootstrap = bootstrap
    return seen


def weights(model, cust):
    return np.stack([cust.decrypt(pm.payload).values for pm in outputs(model)])


def time_reference_step(batches=(1, 2)) -> dict:
    """The reference CkksBackend (numpy, this host) on the c1 shape at small
    batches: per-sample cost = slope, update + refresh = intercept, extrapolated
    to the configured batch of 32 (each sample's pipeline is independent until
    the depth-free delta-W fold, nn.py:363-382)."""
    import_reference()
    import ciphermlp.ckks.backend as rb

    if rb.CkksBackend.__module__ != "ciphermlp.ckks.backend":
        raise RuntimeError("the reference CkksBackend is swapped out; uninstall the plugin")
    secs = {}
    for b in batches:
        cust, model, shape, x, onehot = build(batch=b)
        t0 = time.perf_counter()
        step(cust, model, shape, x, onehot)
        secs[b] = time.perf_counter() - t0
    b0, b1 = min(batches), max(batches)
    slope = (secs[b1] - secs[b0]) / (b1 - b0)
    intercept = secs[b0] - slope * b0
    return {"seconds": secs, "per_sample_s": slope, "update_refresh_s": intercept,
            "ms_per_step_batch32": 1e3 * (intercept + 32 * slope), "cores": 1,
            "kind": "reference",
            "sample": f"unmodified reference CkksBackend (numpy, its own sub-2^31 prime layout: "
                      f"18+2 limbs) running prepare_sample + nn.train_iteration at the config-1 "
                      f"shape with batch {b0} and {b1} on this host; batch-32 step = update/"
                      f"refresh intercept + 32 x per-sample slope"}
