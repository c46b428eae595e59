"""GPU parity: the sm_100a kernels through the C-ABI and the HE API against the
reference's golden vectors (tests/golden, made by the real reference) and the
CPU oracle (oracle/ckks_oracle.py, itself pinned to those vectors).

Integer work must be bit-exact; float encode/decode within 1e-6 per slot
(BASELINE north_star) and the reference's own decrypt tolerances.
"""

import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import ckks_oracle as O  # noqa: E402
from paper_2506_19693_b200 import he_api, he_errors  # noqa: E402
from paper_2506_19693_b200.backend import B200Backend, GpuCiphertext  # noqa: E402
from paper_2506_19693_b200.ring import GpuChain  # noqa: E402
from paper_2506_19693_b200.scheme import SchemeParams, make_params  # noqa: E402


def _u64(t):
    return t.cpu().numpy().astype(np.uint64)


# ---------------------------------------------------------------------------
# NTT (K1) vs reference NttPlan vectors and the oracle
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def ntt_gold(golden_dir):
    return np.load(os.path.join(golden_dir, "ref_ntt.npz"))


def _single_prime_chain(n, p):
    """A GpuChain whose only ciphertext prime is p (tables for NTT tests)."""

    class P:
        poly_degree = n
        modulus_chain = (30, 30, 30)
        scale_bits = 30
        level = 1

    ch = GpuChain.__new__(GpuChain)
    from paper_2506_19693_b200 import _native as nat

    ch.params = P
    ch.layout = "custom"
    ch.n = n
    ch.log_n = n.bit_length() - 1
    ch.device = torch.device("cuda")
    ch.all_primes = [int(p)]
    ch.primes = [int(p)]
    ch.special_primes = []
    ch.lq, ch.k = 1, 0
    mods, ntt, pair = nat.build_tables(ch.log_n, ch.all_primes)
    ch._mods = torch.from_numpy(mods).cuda()
    ch._ntt = torch.from_numpy(ntt.reshape(-1)).cuda()
    ch._pair = torch.from_numpy(pair.reshape(-1)).cuda()
    ch.ring = nat.CkbRing(ch.log_n, 1, ch._mods.data_ptr(), ch._ntt.data_ptr(), ch._pair.data_ptr())
    ch.ring_p = nat.ctypes.pointer(ch.ring)
    ch._maps = {}
    return ch


@pytest.mark.parametrize("n", [16, 64, 1024, 4096, 8192])
def test_ntt_matches_reference_vectors(ntt_gold, n):
    p = int(ntt_gold[f"n{n}_p"][0])
    ch = _single_prime_chain(n, p)
    a = torch.from_numpy(ntt_gold[f"n{n}_in"].astype(np.uint64)).cuda()
    f = ch.ntt_fwd(a.clone(), 1)
    assert np.array_equal(_u64(f), ntt_gold[f"n{n}_fwd"])
    i = ch.ntt_inv(a.clone(), 1)
    assert np.array_equal(_u64(i), ntt_gold[f"n{n}_inv"])


@pytest.mark.parametrize("logn", [5, 10, 12, 13, 14, 15, 16, 17])
@pytest.mark.parametrize("bits", [30, 40, 60])
def test_ntt_big_primes_vs_oracle_and_roundtrip(logn, bits):
    n = 1 << logn
    p = O.largest_ntt_prime_below(bits, 2 * n, set())
    ch = _single_prime_chain(n, p)
    rng = np.random.default_rng(logn * 100 + bits)
    rows = 3
    a_np = rng.integers(0, p, (rows, n), dtype=np.uint64)
    a = torch.from_numpy(a_np).cuda()
    f = ch.ntt_fwd(a.clone(), 1)
    if n <= 4096:  # oracle (object arithmetic) is slow beyond this
        plan = O.NttPlan(p, n)
        want = np.array([int(v) for v in plan.forward(a_np[0])], dtype=np.uint64)
        assert np.array_equal(_u64(f)[0], want)
    back = ch.ntt_inv(f.clone(), 1)
    assert np.array_equal(_u64(back), a_np)
    assert int(_u64(f).max()) < p


@pytest.mark.parametrize("bits0", [60, 40])
@pytest.mark.parametrize("logn", [12, 14, 16])
def test_ntt_out_of_place_matches_in_place(logn, bits0):
    """ckb_ntt_{forward,inverse}_from on a strided component view (items of
    [3][m][N]; FP64-path and integer-path primes mixed, or FP64-path primes
    only: the column-mapped first phase reads the source directly) equals the
    in-place transform of a contiguous copy, and leaves the source untouched."""
    n = 1 << logn
    params = SchemeParams(poly_degree=n, modulus_chain=(bits0, 40, 40, 60), scale_bits=40, level=2)
    ch = GpuChain(params, layout="baseline")
    m, b = 3, 5
    rng = np.random.default_rng(logn)
    x_np = np.stack([np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64)
                                         for p in ch.all_primes[:m]]) for _ in range(3)])
                     for _ in range(b)])
    x = torch.from_numpy(x_np).cuda()
    for inverse in (False, True):
        got = ch.ntt_from(x[:, 1], b, m, 3 * m * n, inverse=inverse)
        want = x[:, 1].contiguous()
        (ch.ntt_inv if inverse else ch.ntt_fwd)(want, m)
        assert torch.equal(got, want)
    assert np.array_equal(_u64(x), x_np)


def test_pt_mac_equals_mul_add_chain():
    """ckb_pt_mac (the BSGS row of bootstrapping) equals the mul_pt / add_ct
    chain it replaces, bit for bit, with terms from x0 and from a stack, and
    the broadcast elementwise kernels equal numpy on odd row counts."""
    n = 1 << 12
    params = SchemeParams(poly_degree=n, modulus_chain=(60, 40, 45, 60), scale_bits=40, level=2)
    ch = GpuChain(params, layout="baseline")
    m, b, nst = 3, 3, 5
    rng = np.random.default_rng(11)
    primes = ch.all_primes[:m]

    def rand(*lead):
        return torch.from_numpy(np.stack([rng.integers(0, p, (*lead, n), dtype=np.uint64)
                                          for p in primes], axis=-2)).cuda()

    x0 = rand(b, 2)
    stack = rand(nst, b, 2)
    idx = [-1, 3, 0, 4, 4, -1, 1]
    pts = rand(len(idx))
    got = ch.pt_mac(x0, stack, idx, pts, m)
    want = None
    for t, k in enumerate(idx):
        term = ch.mul(x0 if k < 0 else stack[k], pts[t], m, b_rows=m)
        want = term if want is None else ch.add(want, term, m)
    assert torch.equal(got, want)
    # elementwise against numpy (object ints): mul with a broadcast plaintext
    a_np, p_np = _u64(x0[0]), _u64(pts[0])
    prod = _u64(ch.mul(x0[0], pts[0], m, b_rows=m))
    for c in range(2):
        for j, p in enumerate(primes):
            w = (a_np[c, j].astype(object) * p_np[j].astype(object)) % p
            assert np.array_equal(prod[c, j], w.astype(np.uint64))
    s_, b_np = _u64(ch.sub(x0[1], x0[0], m)), _u64(x0[1])
    for c in range(2):
        for j, p in enumerate(primes):
            w = (b_np[c, j].astype(object) - a_np[c, j].astype(object)) % p
            assert np.array_equal(s_[c, j], w.astype(np.uint64))


def test_scalar_mac_equals_scalar_mul_chain():
    """ckb_scalar_mac (Chebyshev leaves): sum_k a_k X_k with signed big-int
    scalars and operands at higher levels read restricted, equals numpy."""
    n = 1 << 10
    params = SchemeParams(poly_degree=n, modulus_chain=(60, 40, 45, 60, 60), scale_bits=40,
                          level=3)
    ch = GpuChain(params, layout="baseline")
    rng = np.random.default_rng(5)
    m = 3
    xs_np, xs = [], []
    for mk in (3, 4, 4, 3):  # limbs per poly of each term (>= m)
        a = np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64)
                                for p in ch.all_primes[:mk]]) for _ in range(2 * 2)])
        xs_np.append(a.reshape(2, 2, mk, n))
        xs.append(torch.from_numpy(a.reshape(2, 2, mk, n)).cuda())
    ints = [3, -(1 << 70) + 5, 0, (1 << 90) + 12345]
    got = _u64(ch.scalar_mac(xs, ch.scalar_table(ints, m), m))
    for j, p in enumerate(ch.all_primes[:m]):
        want = sum((x[:, :, j].astype(object) * (a % p)) for x, a in zip(xs_np, ints)) % p
        assert np.array_equal(got[:, :, j], want.astype(np.uint64))


def test_ntt_product_matches_schoolbook_60bit():
    n = 32
    p = O.largest_ntt_prime_below(60, 2 * n, set())
    ch = _single_prime_chain(n, p)
    rng = np.random.default_rng(3)
    a_np = rng.integers(0, p, n, dtype=np.uint64)
    b_np = rng.integers(0, p, n, dtype=np.uint64)
    fa = ch.ntt_fwd(torch.from_numpy(a_np).cuda(), 1)
    fb = ch.ntt_fwd(torch.from_numpy(b_np).cuda(), 1)
    prod = ch.ntt_inv(ch.mul(fa, fb, 1), 1)
    want = O.schoolbook_negacyclic([int(v) for v in a_np], [int(v) for v in b_np], p)
    assert [int(v) for v in _u64(prod)] == want


# ---------------------------------------------------------------------------
# Mode A: the backend against the reference's ciphertext planes
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def ck_gold(golden_dir):
    return np.load(os.path.join(golden_dir, "ref_ckks_n512.npz"))


@pytest.fixture(scope="module")
def mode_a(ck_gold):
    n, level, sb = (int(v) for v in ck_gold["params"])
    params = SchemeParams(poly_degree=n, modulus_chain=tuple(int(v) for v in ck_gold["chain"]),
                          scale_bits=sb, level=level)
    rots = [int(v) for v in ck_gold["rots"]]
    cust = he_api.keygen(params, rots, backend="ckks", rng_seed=int(ck_gold["rng_seed"][0]))
    return cust


def _wrap(cust, planes, level):
    be = cust.backend
    return be._wrap(be.payload_from_planes(planes, level), level, 0)


def _key_digest(key):
    h = hashlib.sha256()
    d = key.data.cpu().numpy()
    for j in range(d.shape[0]):
        h.update(np.ascontiguousarray(d[j, 0].astype("<u8")).tobytes())
        h.update(np.ascontiguousarray(d[j, 1].astype("<u8")).tobytes())
    return h.hexdigest()


def test_mode_a_chain_secret_and_keys_bit_exact(ck_gold, mode_a):
    be = mode_a.backend
    assert be.chain.all_primes == [int(v) for v in ck_gold["all_primes"]]
    assert be.chain.level_limbs == [int(v) for v in ck_gold["level_limbs"]]
    assert np.array_equal(be.sk.coeffs, ck_gold["secret"].astype(np.int64))
    digests = json.loads(str(ck_gold["key_digests"]))
    assert _key_digest(be.relin_key) == digests["relin"]
    for g, key in be.rotation_keys.items():
        assert _key_digest(key) == digests[f"rot_{g}"]


def test_mode_a_ciphertext_ops_bit_exact(ck_gold, mode_a):
    cust = mode_a
    ev = cust.evaluator
    lvl = int(ck_gold["params"][1])
    ct1 = _wrap(cust, ck_gold["ct1"], lvl)
    ct2 = _wrap(cust, ck_gold["ct2"], lvl)
    mul = ev.mul(ct1, ct2)
    deep = ev.mul(mul, ct2)
    got = {
        "add": ev.add(ct1, ct2), "sub": ev.sub(ct1, ct2), "mul": mul,
        "rot1": ev.rotate(ct1, 1), "rot3": ev.rotate(ct1, 3), "rotm1": ev.rotate(ct1, -1),
        "deep": deep, "mixed": ev.add(deep, ct1), "sq": ev.mul(mul, mul),
    }
    for name, cv in got.items():
        assert cv.level_remaining == int(ck_gold[f"lvl_{name}"][0]), name
        assert np.array_equal(cust.backend.planes_of(cv.payload), ck_gold[f"out_{name}"]), name
        dec = cust.decrypt(cv).values
        assert np.max(np.abs(dec - ck_gold[f"dec_{name}"])) <= 1e-6, name


def test_mode_a_plaintext_ops_bit_exact_given_encoding(ck_gold, mode_a):
    """mul_pt/add_pt/sub_pt: the device encoding (cuFFT) may differ from numpy's
    by +-1 in a coefficient; the integer path is checked bit-exactly against the
    oracle fed the device's own encoding, and the encoding within +-1."""
    cust = mode_a
    be = cust.backend
    ev = cust.evaluator
    lvl = int(ck_gold["params"][1])
    n = be.n
    orc = O.OracleCkks(n, tuple(int(v) for v in ck_gold["chain"]), 40, lvl,
                       rotation_steps=[], rng_seed=int(ck_gold["rng_seed"][0]))
    ct1 = _wrap(cust, ck_gold["ct1"], lvl)
    o_ct1 = O.ct_from_u64(ck_gold["ct1"], lvl, orc.chain)
    v3 = ck_gold["v3"]
    pv = he_api.make_plain(v3, n // 2, 40.0)
    dev_c = be.encoder.embed(v3, be.chain.scale_at[lvl])
    assert np.max(np.abs(dev_c - ck_gold["pt3_coeffs"])) <= 1
    dev_cn = be.encoder.embed(-v3, be.chain.scale_at[lvl])
    m3 = O.make_element(orc.chain.limbs_at(lvl), dev_c)
    m3n = O.make_element(orc.chain.limbs_at(lvl), dev_cn)
    cases = {
        "mul_pt": (ev.mul(ct1, pv), orc.mul_plain_coeffs(o_ct1, m3)),
        "add_pt": (ev.add(ct1, pv), orc.add_plain_coeffs(o_ct1, m3)),
        "sub_pt": (ev.sub(ct1, pv), orc.add_plain_coeffs(o_ct1, m3n)),
    }
    for name, (cv, oct_) in cases.items():
        assert np.array_equal(be.planes_of(cv.payload), O.ct_to_u64(oct_, orc.chain)), name
        dec = cust.decrypt(cv).values
        assert np.max(np.abs(dec - ck_gold[f"dec_{name}"])) <= 2.0**-25, name


def test_mode_a_encrypt_bit_exact_given_encoding(ck_gold, mode_a):
    be = mode_a.backend
    lvl = int(ck_gold["params"][1])
    orc = O.OracleCkks(be.n, tuple(int(v) for v in ck_gold["chain"]), 40, lvl,
                       rng_seed=int(ck_gold["rng_seed"][0]))
    # a fresh backend so the serial counter starts where the fixture's did
    cust = he_api.keygen(be.params, [], backend="ckks", rng_seed=int(ck_gold["rng_seed"][0]))
    v1 = ck_gold["v1"]
    cv = cust.encrypt(he_api.make_plain(v1, be.n // 2, 40.0))
    coeffs = cust.backend.encoder.embed(v1, be.chain.scale_at[lvl])
    m = O.make_element(orc.chain.limbs_at(lvl), coeffs)
    want = orc.encrypt_coeffs(m, lvl, int(ck_gold["ct1_serial"][0]) + 1)
    assert np.array_equal(cust.backend.planes_of(cv.payload), O.ct_to_u64(want, orc.chain))
    assert np.max(np.abs(cust.decrypt(cv).values - ck_gold["dec_ct1"])) <= 1e-6


def test_rbct_roundtrip_and_errors(ck_gold, mode_a):
    be = mode_a.backend
    lvl = int(ck_gold["params"][1])
    cv = _wrap(mode_a, ck_gold["ct1"], lvl)
    blob = be.serialize_cipher(cv)
    assert blob[:4] == b"RBCT"
    back = be.deserialize_cipher(blob)
    assert np.array_equal(be.planes_of(back.payload), ck_gold["ct1"])
    with pytest.raises(he_errors.SerializationError):
        be.deserialize_cipher(b"XXXX" + blob[4:])
    with pytest.raises(he_errors.SerializationError):
        be.deserialize_cipher(blob[:-8])


def test_rbct_bytes_identical_to_reference(ck_gold, mode_a):
    """serialize_cipher (ckks/backend.py:210-218) byte for byte, and the
    reference's blobs deserialize to its planes (fresh and post-multiply)."""
    be = mode_a.backend
    for name, lvl_key in (("ct1", None), ("mul", "lvl_mul")):
        planes = ck_gold["ct1"] if name == "ct1" else ck_gold["out_mul"]
        lvl = int(ck_gold["params"][1]) if lvl_key is None else int(ck_gold[lvl_key][0])
        ref_blob = ck_gold[f"rbct_{name}"].tobytes()
        assert be.serialize_cipher(_wrap(mode_a, planes, lvl)) == ref_blob
        back = be.deserialize_cipher(ref_blob)
        assert back.level_remaining == lvl
        assert np.array_equal(be.planes_of(back.payload), planes)


def test_rbky_reference_key_file_round_trip(ck_gold):
    """The reference's RBKY key container (ckks/backend.py:250-293) loads into
    the B200 backend: same secret, bit-identical regenerated keys, and
    save_custodian writes the same bytes back."""
    from paper_2506_19693_b200.backend import load_custodian, save_custodian

    blob = ck_gold["rbky"].tobytes()
    cust = load_custodian(blob)
    be = cust.backend
    assert np.array_equal(be.sk.coeffs, ck_gold["secret"].astype(np.int64))
    digests = json.loads(str(ck_gold["key_digests"]))
    assert _key_digest(be.relin_key) == digests["relin"]
    for g, key in be.rotation_keys.items():
        assert _key_digest(key) == digests[f"rot_{g}"]
    assert save_custodian(cust) == blob
    with pytest.raises(he_errors.SerializationError):
        load_custodian(b"XXXX" + blob[4:])


# ---------------------------------------------------------------------------
# Mode B: BASELINE-style single 40/60-bit primes, hybrid key switching
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("dnum,level,special", [(None, 3, 60), (2, 3, 120), (3, 5, 300),
                                                  (1, 3, 240), (3, 5, 360), (2, 3, 660)])
def test_mode_b_ops_bit_exact_vs_oracle(dnum, level, special):
    """(3, 5, 300): 5 special primes, so ModDown with the fused rescale drops
    5 + 1 primes (k_divround_corr<6, 1>)."""
    n = 256
    chain = (60,) + (40,) * level + (special,)
    params = SchemeParams(poly_degree=n, modulus_chain=chain, scale_bits=40, level=level)
    cust = he_api.keygen(params, {1, 5}, backend="ckks", rng_seed=7, prime_layout="baseline",
                         dnum=dnum, sampler="numpy")  # the oracle's key stream
    be = cust.backend
    alpha = be.alpha
    orc = O.OracleCkks(n, chain, 40, level, rotation_steps=[1, 5], rng_seed=7, layout="baseline",
                       alpha=alpha)
    assert be.chain.all_primes == orc.chain.all_primes
    assert be.relin_key.data.shape[0] == len(orc.relin.rows_b)
    rng = np.random.default_rng(1)
    planes = []
    for _ in range(2):
        c = np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64)
                                for p in orc.chain.limbs_at(level)]) for _ in range(2)])
        planes.append(c)
    ev = cust.evaluator
    a, b = (_wrap(cust, p, level) for p in planes)
    oa, ob = (O.ct_from_u64(p, level, orc.chain) for p in planes)
    o_mul = orc.mul(oa, ob)
    checks = [
        (ev.mul(a, b), o_mul),
        (ev.rotate(a, 1), orc.rotate(oa, 1)),
        (ev.rotate(b, 5), orc.rotate(ob, 5)),
        (ev.add(ev.mul(a, b), a), orc.add(o_mul, oa)),
        (ev.mul(ev.mul(a, b), b), orc.mul(o_mul, ob)),
    ]
    for cv, oct_ in checks:
        assert np.array_equal(be.planes_of(cv.payload), O.ct_to_u64(oct_, orc.chain))
    # fused rotate-and-accumulate (ckb_divround_ntt_combine_acc), batched:
    # a + rot(a, 5) and b + rot(b, 5) in one key switch
    g = pow(5, 5, 2 * n)
    x = torch.stack([a.payload.data, b.payload.data])
    acc = be._hrot(x, level, galois=g, key=be.rotation_key(g), accumulate=True)
    for j, (ct, oct_) in enumerate(((a, oa), (b, ob))):
        want = O.ct_to_u64(orc.add(oct_, orc.rotate(oct_, 5)), orc.chain)
        assert np.array_equal(be.planes_of(GpuCiphertext(acc[j], level)), want)
    # inputs are never modified by an op (CipherVector immutability, api.py:51-65)
    assert np.array_equal(be.planes_of(a.payload), planes[0])
    assert np.array_equal(be.planes_of(b.payload), planes[1])


def test_moddown_fast_conversion_paths_agree():
    """Wide ModDown drops (>= 6 special primes) take the fast basis-conversion
    correction; its exact-rho path (every coefficient forced through it with
    margin 0), its default path and the mixed-radix kernel (use_hps off) give
    the same ciphertexts bit for bit, for HMult (drop + fused rescale) and
    HRot (drop only)."""
    from paper_2506_19693_b200 import _native as nat
    from paper_2506_19693_b200.ring import GpuChain as GC

    n, level = 1024, 4
    chain = (60,) + (40,) * level + (660,)
    params = SchemeParams(poly_degree=n, modulus_chain=chain, scale_bits=40, level=level)
    cust = he_api.keygen(params, {3}, backend="ckks", rng_seed=9, prime_layout="baseline",
                         dnum=2)
    be = cust.backend
    assert be.chain.k == 11
    rng = np.random.default_rng(2)
    planes = [np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64)
                                  for p in be.chain.limbs_at(level)]) for _ in range(2)])
              for _ in range(2)]
    a, b = (_wrap(cust, p, level) for p in planes)
    ev = cust.evaluator

    def run():
        return (be.planes_of(ev.mul(a, b).payload), be.planes_of(ev.rotate(a, 3).payload))

    base = run()
    try:
        be.chain.set_ring_flag(nat.RING_HPS_EXACT, True)
        forced = run()
    finally:
        be.chain.set_ring_flag(nat.RING_HPS_EXACT, False)
    GC.use_hps = False
    try:
        chained = run()
    finally:
        GC.use_hps = True
    for x, y, z in zip(base, forced, chained):
        assert np.array_equal(x, y) and np.array_equal(x, z)


def test_low_special_modulus_keyswitch():
    """Level-aware special modulus (low_special): at or below the refresh level
    multiplies and rotations key-switch over Q u P' (first k' special primes)
    and decrypt like the full-P key switch; above it the full P is used, and
    a P' narrower than a digit is rejected."""
    n, L, bd = 1 << 10, 6, 2
    chain = (60,) + (45,) * (L - bd) + (60,) * bd + (360,)
    params = SchemeParams(poly_degree=n, modulus_chain=chain, scale_bits=45, level=L,
                          bootstrap_depth=bd)
    opts = dict(backend="ckks", rng_seed=3, prime_layout="bootstrap", dnum=3, secret_hw=64)
    full = he_api.keygen(params, {1}, **opts)
    low = he_api.keygen(params, {1}, low_special=4, **opts)
    assert low.backend.k_low == 4 and full.backend.k_low is None
    rl = params.refresh_level
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, n // 2)
    w = rng.uniform(-1, 1, n // 2)
    for cust in (full, low):
        be = cust.backend
        a = cust.encrypt(he_api.make_plain(v, n // 2, 45.0))
        b = cust.encrypt(he_api.make_plain(w, n // 2, 45.0))
        ev = cust.evaluator
        # bring both to the refresh level, then multiply and rotate there
        while a.level_remaining > rl:
            a = ev.mul(a, cust.encrypt(he_api.make_plain(np.ones(n // 2), n // 2, 45.0)))
            b = ev.mul(b, cust.encrypt(he_api.make_plain(np.ones(n // 2), n // 2, 45.0)))
        assert be._low(a.level_remaining) == (cust is low)
        prod = cust.decrypt(ev.mul(a, b)).values
        rot = cust.decrypt(ev.rotate(a, 1)).values
        assert np.max(np.abs(prod - v * w)) < 1e-6
        assert np.max(np.abs(rot - np.roll(v, -1))) < 1e-6
    with pytest.raises(Exception):
        he_api.keygen(params, {1}, low_special=1, **opts)


def test_low_special_two_tiers_pick_k_per_level():
    """low_special as a tier list (what the config-4/5 runs use): each level
    picks the k' of the first tier covering it (full P above the last tier),
    results decrypt correctly at every level, numpy integers are accepted and
    out-of-range tiers are rejected."""
    n, L, bd = 1 << 10, 6, 2
    chain = (60,) + (45,) * (L - bd) + (60,) * bd + (360,)
    params = SchemeParams(poly_degree=n, modulus_chain=chain, scale_bits=45, level=L,
                          bootstrap_depth=bd)
    opts = dict(backend="ckks", rng_seed=3, prime_layout="bootstrap", dnum=3, secret_hw=64)
    cust = he_api.keygen(params, {1}, low_special=[(np.int64(2), 3), (4, np.int32(4))], **opts)
    be = cust.backend
    assert [be._ks_k(lv) for lv in range(L + 1)] == [3, 3, 3, 4, 4, 6, 6]
    rng = np.random.default_rng(1)
    v = rng.uniform(-1, 1, n // 2)
    a = cust.encrypt(he_api.make_plain(v, n // 2, 45.0))
    ev = cust.evaluator
    want = v.copy()
    one = he_api.make_plain(np.ones(n // 2), n // 2, 45.0)
    while a.level_remaining > 0:
        r = ev.rotate(a, 1)
        assert np.max(np.abs(cust.decrypt(r).values - np.roll(want, -1))) < 1e-6
        a = ev.mul(a, cust.encrypt(one))
        assert np.max(np.abs(cust.decrypt(a).values - want)) < 1e-6
    for bad in ([(2, 6)], [(2, 0)], [(9, 3)], "x"):
        with pytest.raises(he_errors.InvalidParameters):
            he_api.keygen(params, {1}, low_special=bad, **opts)


# ---------------------------------------------------------------------------
# Decryption tolerances (tests/test_ckks_backend.py of the reference)
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def ckks_small():
    params = make_params(level=10, scale_bits=40, poly_degree=2**12)
    return params, he_api.keygen(params, {1, 2, 3, -1}, backend="ckks", rng_seed=0)


def _pl(cust, v):
    return he_api.make_plain(v, cust.params.slot_count, float(cust.params.scale_bits))


def test_encode_roundtrip_and_overflow(ckks_small):
    params, cust = ckks_small
    be = cust.backend
    v = np.random.default_rng(9).uniform(-1, 1, params.slot_count)
    c = be.encoder.embed(v, 2.0**40)
    assert np.max(np.abs(be.encoder.unembed(c.astype(np.float64), 2.0**40) - v)) <= 2.0**-30
    ref = O.Encoder(params.poly_degree).embed(v, 2.0**40)
    assert np.max(np.abs(c - ref)) <= 1
    assert np.max(np.abs(be.encoder.unembed(c.astype(np.float64), 2.0**40)
                         - O.Encoder(params.poly_degree).unembed(c, 2.0**40))) <= 1e-6
    with pytest.raises(he_errors.EncodingOverflow):
        cust.encrypt(_pl(cust, np.full(params.slot_count, 2.0**25)))


def test_homomorphic_ops_within_tolerance(ckks_small):
    params, cust = ckks_small
    ev = cust.evaluator
    rng = np.random.default_rng(23)
    for _ in range(5):
        a = rng.uniform(-1, 1, params.slot_count)
        b = rng.uniform(-1, 1, params.slot_count)
        ca, cb = cust.encrypt(_pl(cust, a)), cust.encrypt(_pl(cust, b))
        assert np.max(np.abs(cust.decrypt(ca).values - a)) <= 2.0**-30
        for got, want in [(ev.add(ca, cb), a + b), (ev.sub(ca, cb), a - b), (ev.mul(ca, cb), a * b),
                          (ev.mul(ca, _pl(cust, b)), a * b), (ev.add(ca, _pl(cust, b)), a + b),
                          (ev.rotate(ca, 1), np.roll(a, -1)), (ev.rotate(ca, -1), np.roll(a, 1))]:
            assert np.max(np.abs(cust.decrypt(got).values - want)) <= 2.0**-25


def test_multiply_chain_level_exhaustion_and_bootstrap(ckks_small):
    params, cust = ckks_small
    ev = cust.evaluator
    x = cust.encrypt(_pl(cust, np.full(params.slot_count, 0.9)))
    ones = cust.encrypt(_pl(cust, np.ones(params.slot_count)))
    for _ in range(10):
        x = ev.mul(x, ones)
    assert x.level_remaining == 0
    with pytest.raises(he_errors.LevelExhausted):
        ev.mul(x, ones)
    before = cust.decrypt(x).values
    assert np.max(np.abs(before - 0.9)) <= 2.0**-20
    r = cust.bootstrap(x)
    assert r.level_remaining == params.refresh_level
    assert np.max(np.abs(cust.decrypt(r).values - before)) <= 2.0**-28


def test_missing_rotation_key(ckks_small):
    params, cust = ckks_small
    ct = cust.encrypt(_pl(cust, np.zeros(params.slot_count)))
    with pytest.raises(he_errors.MissingRotationKey):
        cust.evaluator.rotate(ct, 5)


# ---------------------------------------------------------------------------
# Config-2 sizes: N=2^16, 40-bit limbs, dnum=3 (size-independent properties)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("L", [4, 12])
def test_c2_hybrid_keyswitch_decrypts(L):
    k = {4: 2, 12: 3, 24: 6}[L]
    params = make_params(level=L - 1, scale_bits=40, poly_degree=2**16, first_bits=40,
                         special_bits=60 * k)
    cust = he_api.keygen(params, {1, 7}, backend="ckks", rng_seed=2, prime_layout="baseline",
                         dnum=3, secret_hw=192)
    be = cust.backend
    assert be.chain.k == k and be.alpha == -(-L // 3)
    ev = cust.evaluator
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, params.slot_count)
    b = rng.uniform(-1, 1, params.slot_count)
    ca, cb = cust.encrypt(_pl(cust, a)), cust.encrypt(_pl(cust, b))
    assert np.max(np.abs(cust.decrypt(ev.mul(ca, cb)).values - a * b)) <= 2.0**-20
    assert np.max(np.abs(cust.decrypt(ev.rotate(ca, 7)).values - np.roll(a, -7))) <= 2.0**-20


# ---------------------------------------------------------------------------
# Config-1 step: the reference train_iteration's HE calls, replayed
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def c1_program(golden_dir):
    from paper_2506_19693_b200.replay import Program

    path = os.path.join(golden_dir, "c1_trace.npz")
    return Program.load(path), np.load(path)


def _c1_custodian(z):
    n, level, sb = (int(v) for v in z["params"])
    params = make_params(level=level, scale_bits=sb, poly_degree=n)
    return he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3,
                         prime_layout="baseline", secret_hw=64)


def test_c1_step_weights_match_reference(c1_program):
    """Decrypted weights/velocities after one encrypted step agree with the
    reference CKKS run and the exact float model within 1e-3 (north_star)."""
    prog, z = c1_program
    cust = _c1_custodian(z)
    env = prog.run(cust)
    w = np.stack([cust.decrypt(env[o]).values for o in prog.outputs])
    assert np.max(np.abs(w - z["sim_weights"])) <= 1e-3
    if "ckks_weights" in z:
        assert np.max(np.abs(w - z["ckks_weights"])) <= 1e-3


def test_wave_executor_bit_identical_to_sequential(c1_program):
    from paper_2506_19693_b200.executor import WaveExecutor

    prog, z = c1_program
    seq = _c1_custodian(z)
    env_seq = prog.run(seq)
    bat = _c1_custodian(z)
    env_bat = WaveExecutor(prog, bat).run()
    for o in prog.outputs:
        a = seq.backend.planes_of(env_seq[o].payload)
        b = bat.backend.planes_of(env_bat[o])
        assert np.array_equal(a, b)


def test_graphed_step_bit_identical_to_eager(c1_program):
    """graphs.GraphedStep: the config-1 step captured as one CUDA graph (the
    refreshes eager afterwards) reproduces the eager executor bit for bit, on
    every replay, each replay with its own encryption serials."""
    from paper_2506_19693_b200.executor import WaveExecutor
    from paper_2506_19693_b200.graphs import GraphedStep

    prog, z = c1_program
    cust = _c1_custodian(z)
    env = prog.run(cust, 0, prog.n_setup)
    from paper_2506_19693_b200.graphs import eager_equivalent

    ex = WaveExecutor(prog, cust)
    gs = GraphedStep(ex, env)
    prev = None
    for _ in range(2):
        got_env = gs.step()
        got = [cust.backend.planes_of(got_env[o]) for o in prog.outputs]
        want_env = eager_equivalent(gs)
        want = [cust.backend.planes_of(want_env[o]) for o in prog.outputs]
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
        # every replay encrypts with fresh randomness (its own serials)
        assert prev is None or not all(np.array_equal(a, b) for a, b in zip(got, prev))
        prev = got


# ---------------------------------------------------------------------------
# Config 3: homomorphic bootstrapping (no reference counterpart: parity
# unpinned; the check is decrypt(bootstrap(ct)) against the input values)
# ---------------------------------------------------------------------------


def test_real_bootstrap_precision_n8192():
    n, L = 1 << 13, 24
    params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,),
                          scale_bits=45, level=L, bootstrap_depth=16)
    cust = he_api.keygen(params, {1}, backend="ckks", rng_seed=1, prime_layout="bootstrap",
                         dnum=3, secret_hw=192, real_bootstrap=True)
    be = cust.backend
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, n // 2)
    ct = cust.encrypt(he_api.make_plain(v, n // 2, 45.0))
    # consume levels, then refresh through the HE API
    ct = cust.evaluator.mul(ct, he_api.make_plain(np.ones(n // 2), n // 2, 45.0))
    r = cust.bootstrap(ct)
    assert r.level_remaining == params.refresh_level
    err = np.max(np.abs(cust.decrypt(r).values - v))
    assert err <= 2.0**-15, err
    # the refreshed ciphertext keeps computing
    sq = cust.evaluator.mul(r, r)
    assert np.max(np.abs(cust.decrypt(sq).values - v * v)) <= 2.0**-14


def test_batched_bootstrap_equals_single():
    """backend.bootstrap_batch (all stages once over a batch, used for the
    refreshes of a training step) gives each ciphertext's single bootstrap
    bit for bit."""
    n, L = 1 << 13, 24
    params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,),
                          scale_bits=45, level=L, bootstrap_depth=16)
    cust = he_api.keygen(params, {1}, backend="ckks", rng_seed=2, prime_layout="bootstrap",
                         dnum=3, secret_hw=192, real_bootstrap=True)
    be = cust.backend
    rng = np.random.default_rng(1)
    vals = [rng.uniform(-1, 1, n // 2) for _ in range(3)]
    cts = [be._encrypt_values(v, 3) for v in vals]
    single = [be.bootstrap_ct(c).data for c in cts]
    batch = be.bootstrap_batch(torch.stack([c.data for c in cts]), 3)
    for j in range(3):
        assert torch.equal(batch[j].view(torch.int64), single[j].view(torch.int64))
    from paper_2506_19693_b200.backend import GpuCiphertext

    rl = params.refresh_level
    err = max(float(np.max(np.abs(be._decrypt_values(GpuCiphertext(batch[j], rl)) - vals[j])))
              for j in range(3))
    assert err <= 2.0**-15


def test_philox_sampler_distribution_and_batch_determinism():
    """ckb_sample: uniform residues in [0, p), rounded N(0, 3.2^2) errors, one
    stream per seed (batched == one at a time)."""
    params = make_params(level=3, scale_bits=40, poly_degree=4096)
    be = he_api.keygen(params, [], backend="ckks", prime_layout="baseline").backend
    ch = be.chain
    seeds = torch.tensor([11, 22, 33], dtype=torch.int64, device="cuda").view(torch.uint64)
    a, e = ch.sample(seeds, 4)
    a1, e1 = ch.sample(seeds[1:2].clone(), 4)
    assert torch.equal(a[1:2].view(torch.int64), a1.view(torch.int64))
    assert torch.equal(e[1:2], e1)
    an = a.cpu().numpy().astype(np.float64)
    for j, p in enumerate(ch.primes[:4]):
        col = an[:, j]
        assert col.max() < p and abs(col.mean() / p - 0.5) < 0.01
    en = e.cpu().numpy()
    assert abs(en.std() - 3.2) < 0.1 and abs(en.mean()) < 0.1
    assert not torch.equal(a[0].view(torch.int64), a[1].view(torch.int64))
