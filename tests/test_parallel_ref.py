"""The multi-core CPU baseline (oracle/parallel_ref.py) computes exactly the
oracle's (= the reference's) HMult."""

import numpy as np

from oracle import ckks_oracle as O
from oracle import parallel_ref as PR


def test_parallel_hmult_matches_oracle():
    chain, (a, b), kb, ka = PR.make_random_case(256, 3, seed=4)
    o = O.OracleCkks.__new__(O.OracleCkks)
    o.chain, o.n, o.alpha = chain, 256, 1
    o.relin = O.KSKey([kb] * len(chain.primes), [ka] * len(chain.primes))
    want = O.ct_to_u64(o.mul(a, b), chain)
    for procs in (1, 3):
        got, secs = PR.hmult_parallel(chain, a, b, kb, ka, procs)
        assert np.array_equal(O.ct_to_u64(got, chain), want)
        assert secs > 0


def test_parallel_hrot_matches_oracle():
    chain, (a, _), kb, ka = PR.make_random_case(256, 3, seed=6)
    o = O.OracleCkks.__new__(O.OracleCkks)
    o.chain, o.n, o.alpha = chain, 256, 1
    g = pow(5, 3, 512)
    o.rot_keys = {g: O.KSKey([kb] * len(chain.primes), [ka] * len(chain.primes))}
    want = O.ct_to_u64(o.rotate(a, 3), chain)
    for procs in (1, 2):
        got, secs = PR.hrot_parallel(chain, a, g, kb, ka, procs)
        assert np.array_equal(O.ct_to_u64(got, chain), want)
        assert secs > 0
