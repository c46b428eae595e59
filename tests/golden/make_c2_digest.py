"""Golden digests for the config-2 key-switching paths at full size.

Runs the CPU oracle (oracle/ckks_oracle.py, test infrastructure) on the exact
BASELINE config-2 chain structure — N=2^16, L x 40-bit Q primes, dnum=3
(alpha = ceil(L/3)), k = ceil(40 alpha / 60) 60-bit special primes — for one
HMult (ct x ct + relinearise + rescale, ckks/backend.py:136-143) and one HRot
(ckks/backend.py:155-171) of seeded uniform ciphertexts, and records the
SHA-256 of the output planes (coefficient domain, RBCT order).  The GPU test
tests/test_gpu_headline.py::test_c2_full_size_digest rebuilds the same keys
(sampler="numpy", the oracle's key stream) and inputs and compares digests.

    python tests/golden/make_c2_digest.py [L ...]     # default: 4 12 24

Takes minutes per L (object-array arithmetic at N=2^16); run once, commit
tests/golden/c2_digests.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ckks_oracle as O  # noqa: E402

N = 1 << 16
DNUM = 3
ROT_STEP = 12345
KEY_SEED = 21
PLANE_SEED = 31
SECRET_HW = 192


def case(L):
    alpha = -(-L // DNUM)
    k = -(-40 * alpha // 60)
    chain = (40,) * L + (60 * k,)
    return alpha, k, chain


def hw_secret(n, h, seed):
    """Same construction as backend._hw_secret (positions and signs from
    default_rng((seed, 0x5EC7)))."""
    rng = np.random.default_rng((seed, 0x5EC7))
    s = np.zeros(n, dtype=np.int64)
    pos = rng.choice(n, size=h, replace=False)
    s[pos] = rng.choice(np.array([-1, 1], dtype=np.int64), size=h)
    return s


def input_planes(primes, n, seed):
    rng = np.random.default_rng(seed)
    return [np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
                      for _ in range(2)]) for _ in range(2)]


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<u8").tobytes()).hexdigest()


def run(L):
    alpha, k, chain = case(L)
    level = L - 1
    t0 = time.time()
    orc = O.OracleCkks(N, chain, 40, level, rotation_steps=[ROT_STEP], rng_seed=KEY_SEED,
                       layout="baseline", alpha=alpha, secret=hw_secret(N, SECRET_HW, KEY_SEED))
    t1 = time.time()
    pa, pb = input_planes(orc.chain.limbs_at(level), N, PLANE_SEED)
    oa, ob = (O.ct_from_u64(p, level, orc.chain) for p in (pa, pb))
    mul = O.ct_to_u64(orc.mul(oa, ob), orc.chain)
    t2 = time.time()
    rot = O.ct_to_u64(orc.rotate(oa, ROT_STEP), orc.chain)
    t3 = time.time()
    return {"L": L, "alpha": alpha, "k": k, "n": N, "level": level,
            "all_primes": [int(p) for p in orc.chain.all_primes],
            "rot_step": ROT_STEP, "key_seed": KEY_SEED, "plane_seed": PLANE_SEED,
            "secret_hw": SECRET_HW,
            "inputs_sha256": [digest(pa), digest(pb)],
            "hmult_sha256": digest(mul), "hrot_sha256": digest(rot),
            "hmult_shape": list(mul.shape), "hrot_shape": list(rot.shape),
            "oracle_seconds": {"keygen": t1 - t0, "hmult": t2 - t1, "hrot": t3 - t2}}


def main(argv):
    Ls = [int(a) for a in argv] or [4, 12, 24]
    path = os.path.join(HERE, "c2_digests.json")
    out = {}
    if os.path.exists(path):
        with open(path) as fh:
            out = json.load(fh)
    for L in Ls:
        res = run(L)
        print(json.dumps({kk: v for kk, v in res.items() if kk != "all_primes"}), flush=True)
        out[f"L{L}"] = res
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
