"""Pin the CPU oracle (oracle/ckks_oracle.py) against golden vectors produced by
the REAL reference package (tests/golden/make_golden.py): NTT tables/transforms
(ckks/ntt.py:100-154), key generation (ckks/keys.py:49-142) and every
ciphertext operation of ckks/backend.py:124-190, bit for bit."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import ckks_oracle as O


@pytest.fixture(scope="module")
def ntt_gold(golden_dir):
    return np.load(os.path.join(golden_dir, "ref_ntt.npz"))


@pytest.mark.parametrize("n", [16, 64, 1024, 4096, 8192])
def test_oracle_ntt_matches_reference(ntt_gold, n):
    p = int(ntt_gold[f"n{n}_p"][0])
    plan = O.NttPlan(p, n)
    a = ntt_gold[f"n{n}_in"]
    assert np.array_equal(plan.forward(a), ntt_gold[f"n{n}_fwd"])
    assert np.array_equal(plan.inverse(a), ntt_gold[f"n{n}_inv"])
    k = min(n, 64)
    assert np.array_equal(plan.psi_brv[:k].astype(np.uint64), ntt_gold[f"n{n}_psi_brv"])


@pytest.mark.parametrize("n", [16, 32, 64])
def test_oracle_ntt_schoolbook(n):
    # known-answer test of tests/test_ckks_ring.py:48-57
    rng = np.random.default_rng(n)
    p = O.nearest_ntt_prime(1 << 26, 2 * n, set())
    plan = O.NttPlan(p, n)
    for _ in range(4):
        a = rng.integers(0, p, n, dtype=np.uint64)
        b = rng.integers(0, p, n, dtype=np.uint64)
        got = plan.inverse(plan.forward(a) * plan.forward(b) % np.uint64(p))
        assert got.tolist() == O.schoolbook_negacyclic(a.tolist(), b.tolist(), p)


def test_oracle_big_prime_ntt_schoolbook():
    n = 32
    used = set()
    for bits in (40, 60):
        p = O.largest_ntt_prime_below(bits, 2 * n, used)
        plan = O.NttPlan(p, n)
        rng = np.random.default_rng(bits)
        a = [int(v) for v in rng.integers(0, p, n, dtype=np.uint64)]
        b = [int(v) for v in rng.integers(0, p, n, dtype=np.uint64)]
        fa, fb = plan.forward(a), plan.forward(b)
        got = plan.inverse(fa * fb % p)
        assert [int(v) for v in got] == O.schoolbook_negacyclic(a, b, p)
        assert [int(v) for v in plan.inverse(fa)] == a


@pytest.fixture(scope="module")
def ck_gold(golden_dir):
    return np.load(os.path.join(golden_dir, "ref_ckks_n512.npz"))


@pytest.fixture(scope="module")
def ck_oracle(ck_gold):
    n, level, sb = (int(v) for v in ck_gold["params"])
    return O.OracleCkks(n, tuple(int(v) for v in ck_gold["chain"]), sb, level,
                        rotation_steps=[int(v) for v in ck_gold["rots"]],
                        rng_seed=int(ck_gold["rng_seed"][0]), layout="reference")


def _digest(key):
    h = hashlib.sha256()
    for b, a in zip(key.rows_b, key.rows_a):
        h.update(np.ascontiguousarray(b.to_u64().astype("<u8")).tobytes())
        h.update(np.ascontiguousarray(a.to_u64().astype("<u8")).tobytes())
    return h.hexdigest()


def test_oracle_chain_and_keys(ck_gold, ck_oracle):
    ch = ck_oracle.chain
    assert ch.all_primes == [int(v) for v in ck_gold["all_primes"]]
    assert ch.level_limbs == [int(v) for v in ck_gold["level_limbs"]]
    assert np.allclose(ch.scale_at, ck_gold["scale_at"], rtol=0, atol=0)
    assert np.array_equal(ck_oracle.secret, ck_gold["secret"].astype(np.int64))
    digests = json.loads(str(ck_gold["key_digests"]))
    assert _digest(ck_oracle.relin) == digests["relin"]
    for g, key in ck_oracle.rot_keys.items():
        assert _digest(key) == digests[f"rot_{g}"]


def test_oracle_ciphertext_ops_bit_exact(ck_gold, ck_oracle):
    o = ck_oracle
    ch = o.chain
    lvl = o.level
    # encryption: the reference draws default_rng((seed, serial+1)) (api.py:225 + backend.py:174)
    ct1 = o.encrypt(ck_gold["v1"], lvl, int(ck_gold["ct1_serial"][0]) + 1)
    ct2 = o.encrypt(ck_gold["v2"], lvl, int(ck_gold["ct2_serial"][0]) + 1)
    assert np.array_equal(O.ct_to_u64(ct1, ch), ck_gold["ct1"])
    assert np.array_equal(O.ct_to_u64(ct2, ch), ck_gold["ct2"])
    m3 = O.make_element(ch.limbs_at(lvl), ck_gold["pt3_coeffs"])
    m3n = O.make_element(ch.limbs_at(lvl), ck_gold["pt3neg_coeffs"])
    assert np.array_equal(o.encoder.embed(ck_gold["v3"], o.scale(lvl)), ck_gold["pt3_coeffs"])
    n = o.n
    mul = o.mul(ct1, ct2)
    deep = o.mul(mul, ct2)
    got = {
        "add": o.add(ct1, ct2),
        "sub": o.add(ct1, ct2, sub=True),
        "mul": mul,
        "rot1": o.rotate(ct1, 1),
        "rot3": o.rotate(ct1, 3),
        "rotm1": o.rotate(ct1, (-1) % (n // 2)),
        "mul_pt": o.mul_plain_coeffs(ct1, m3),
        "add_pt": o.add_plain_coeffs(ct1, m3),
        "sub_pt": o.add_plain_coeffs(ct1, m3n),
        "deep": deep,
        "mixed": o.add(deep, ct1),
        "sq": o.mul(mul, mul),
    }
    for name, ct in got.items():
        assert ct.level == int(ck_gold[f"lvl_{name}"][0]), name
        assert np.array_equal(O.ct_to_u64(ct, ch), ck_gold[f"out_{name}"]), name
        dec = o.decrypt(ct)
        assert np.max(np.abs(dec - ck_gold[f"dec_{name}"])) <= 1e-12, name
