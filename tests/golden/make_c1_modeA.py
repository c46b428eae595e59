"""Golden digests of one config-1 training step run by the REAL reference.

Runs the unmodified reference (``ciphermlp`` from /root/reference/pkg/src or
baseline/_ref) with its own numpy ``CkksBackend``: keygen (rng_seed 3),
Xavier weights, 32 encrypted samples and ``nn.train_iteration``
(nn.py:344-404) at the config-1 shape (tools/c1_dropin.py), and records the
SHA-256 of the RBCT bytes (ckks/backend.py:210-222: coefficient planes) of

  * the 4 ciphertexts handed to the debug refresh (updated weights and
    velocities, i.e. everything the step computes homomorphically), and
  * the 4 refreshed outputs,

plus their decryptions.  tests/test_gpu_dropin.py runs the same step through
the same reference code with the B200 backend installed (mode A: the
reference prime layout, numpy samplers and numpy FFT encoder) and requires
every digest to match.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c1_modeA.py   # ~3 min
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import c1_dropin as C  # noqa: E402


def main():
    C.import_reference()
    t0 = time.time()
    cust, model, shape, x, onehot = C.build()
    t1 = time.time()
    seen = C.capture_refresh_inputs(cust)
    C.step(cust, model, shape, x, onehot)
    t2 = time.time()
    out = {
        "refresh_inputs_sha256": seen,
        "outputs_sha256": [C.sha(cust.backend.serialize_cipher(pm.payload))
                           for pm in C.outputs(model)],
        "initial_weights_note": "Xavier weights encrypted after keygen (encrypt serials 1..)",
        "seconds": {"build": t1 - t0, "step": t2 - t1},
    }
    np.save(os.path.join(HERE, "c1_modeA_weights.npy"), C.weights(model, cust))
    with open(os.path.join(HERE, "c1_modeA_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out["seconds"]))


if __name__ == "__main__":
    main()
