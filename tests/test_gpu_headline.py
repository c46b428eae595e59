"""GPU parity on the benchmarked configuration's own code paths.

bench.py's headline (BASELINE config 2) runs ``batch_hmult`` (tensor,
alpha = ceil(L/3)-limb ModUp, inner product with the relinearisation key,
ModDown with k special primes fused with the rescale) and ``batch_hrot``
(per-item Galois elements and per-item key pointers) at N=2^16, L x 40-bit
primes, dnum=3, k=ceil(40 alpha/60) 60-bit special primes.  These tests pin
exactly those paths bit for bit against the CPU oracle
(oracle/ckks_oracle.py, itself pinned to the reference's vectors), which
restates ckks/keys.py:74-100 and ckks/backend.py:136-171 with the standard
fast basis conversion for alpha > 1:

  * the exact config-2 chain structure (24 / 12 / 4 limbs, alpha 8 / 4 / 2,
    k 6 / 3 / 2) at N=2^10, with 64 distinct per-item rotation keys at L=24;
  * the N=2^16 single-limb forward and inverse NTT at 40- and 60-bit primes
    (the FP64 and the integer butterfly paths);
  * one N=2^16 HMult and HRot at L = 4, 12, 24 against SHA-256 digests the
    oracle computed on the CPU box (tests/golden/make_c2_digest.py).
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
from paper_2506_19693_b200 import he_api  # noqa: E402
from paper_2506_19693_b200 import _native as nat  # noqa: E402
from paper_2506_19693_b200.ring import GpuChain  # noqa: E402
from paper_2506_19693_b200.scheme import make_params  # noqa: E402

DNUM = 3


def _c2_params(L, n):
    alpha = -(-L // DNUM)
    k = -(-40 * alpha // 60)
    return make_params(level=L - 1, scale_bits=40, poly_degree=n, first_bits=40,
                       special_bits=60 * k), alpha, k


def _planes(primes, n, rng):
    return np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
                     for _ in range(2)])


def _sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<u8").tobytes()).hexdigest()


def _pair(L, n, steps, seed):
    params, alpha, k = _c2_params(L, n)
    cust = he_api.keygen(params, set(steps), backend="ckks", rng_seed=seed,
                         prime_layout="baseline", dnum=DNUM, secret_hw=192,
                         sampler="numpy")  # the oracle's key stream
    be = cust.backend
    assert be.alpha == alpha and be.chain.k == k
    orc = O.OracleCkks(n, params.modulus_chain, 40, params.level, rotation_steps=list(steps),
                       rng_seed=seed, layout="baseline", alpha=alpha, secret=be.sk.coeffs)
    assert be.chain.all_primes == orc.chain.all_primes
    return cust, be, orc


def _to_batch(be, planes_list, level):
    return torch.stack([be.payload_from_planes(p, level).data for p in planes_list])


@pytest.mark.parametrize("L,batch", [(24, 3), (12, 4), (4, 4)])
def test_batch_hmult_config2_structure_bit_exact(L, batch):
    """batch_hmult at alpha = ceil(L/3), k special primes (k_modup_mixed<alpha>,
    the fast-conversion / mixed-radix ModDown with the fused rescale), every
    item bit-exact against OracleCkks.mul."""
    n = 1024
    cust, be, orc = _pair(L, n, [], seed=7)
    lvl = L - 1
    rng = np.random.default_rng(L)
    pa = [_planes(orc.chain.limbs_at(lvl), n, rng) for _ in range(batch)]
    pb = [_planes(orc.chain.limbs_at(lvl), n, rng) for _ in range(batch)]
    out = be.batch_hmult(_to_batch(be, pa, lvl), _to_batch(be, pb, lvl), lvl)
    assert out.shape == (batch, 2, be.chain.level_limbs[lvl - 1], n)
    for i in range(batch):
        oa, ob = (O.ct_from_u64(p, lvl, orc.chain) for p in (pa[i], pb[i]))
        want = O.ct_to_u64(orc.mul(oa, ob), orc.chain)
        got = be.planes_of(_wrap_payload(out[i], lvl - 1))
        assert np.array_equal(got, want), f"item {i}"


def _wrap_payload(data, level):
    from paper_2506_19693_b200.backend import GpuCiphertext

    return GpuCiphertext(data.contiguous(), level)


@pytest.mark.parametrize("L,batch", [(24, 64), (12, 8), (4, 8)])
def test_batch_hrot_per_item_keys_bit_exact(L, batch):
    """batch_hrot with `batch` distinct rotation steps: per-item Galois elements
    (k_automorphism_ntt) and per-item key pointers (the key_ptrs branch of
    k_ks_inner), every item bit-exact against OracleCkks.rotate with its own
    key.  L=24: 64 distinct keys, as in the benchmark."""
    n = 1024
    rng = np.random.default_rng(100 + L)
    steps = [int(s) for s in rng.choice(np.arange(1, n // 2), size=batch, replace=False)]
    cust, be, orc = _pair(L, n, steps, seed=8)
    lvl = L - 1
    pa = [_planes(orc.chain.limbs_at(lvl), n, rng) for _ in range(batch)]
    x = _to_batch(be, pa, lvl)
    g_items, ptrs, keys = be._rotation_tables(steps)
    assert len({k.data.data_ptr() for k in keys}) == batch  # distinct keys per item
    out = be.batch_hrot(x, steps, lvl)
    for i in range(batch):
        want = O.ct_to_u64(orc.rotate(O.ct_from_u64(pa[i], lvl, orc.chain), steps[i]), orc.chain)
        assert np.array_equal(be.planes_of(_wrap_payload(out[i], lvl)), want), f"item {i}"
    # the input batch is never modified
    assert all(np.array_equal(be.planes_of(_wrap_payload(x[i], lvl)), pa[i])
               for i in range(batch))


@pytest.mark.parametrize("inputs", ["random", "extreme"])
@pytest.mark.parametrize("bits", [40, 60])
def test_ntt_n65536_single_limb_bit_exact(bits, inputs):
    """The N=2^16 two-phase transform (forward and inverse) bit-exact against
    the oracle's NttPlan (ntt.py:121-154) on three limbs: 40-bit primes run
    the FP64 butterfly, 60-bit primes the integer one.  "extreme": rows that
    drive the lazy ranges of the butterflies to their bounds (every residue
    p - 1; p - 1 and 0 alternating; p - 1 in the upper half only)."""
    n = 1 << 16
    p = O.largest_ntt_prime_below(bits, 2 * n, set())
    ch = _single_prime_chain(n, p)
    rng = np.random.default_rng(bits)
    if inputs == "random":
        a_np = rng.integers(0, p, (3, n), dtype=np.uint64)
    else:
        a_np = np.zeros((3, n), dtype=np.uint64)
        a_np[0, :] = p - 1
        a_np[1, ::2] = p - 1
        a_np[2, n // 2:] = p - 1
    plan = O.NttPlan(p, n)
    f = ch.ntt_fwd(torch.from_numpy(a_np).cuda(), 1).cpu().numpy()
    inv = ch.ntt_inv(torch.from_numpy(a_np).cuda(), 1).cpu().numpy()
    for r in range(3):
        want_f = np.array([int(v) for v in plan.forward(a_np[r])], dtype=np.uint64)
        want_i = np.array([int(v) for v in plan.inverse(a_np[r])], dtype=np.uint64)
        assert np.array_equal(f[r], want_f), f"forward row {r}"
        assert np.array_equal(inv[r], want_i), f"inverse row {r}"


def _single_prime_chain(n, p):
    """A GpuChain whose only prime is p (NTT tables only)."""
    ch = GpuChain.__new__(GpuChain)
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
    ch.ring = nat.CkbRing(ch.log_n, 1, ch._mods.data_ptr(), ch._ntt.data_ptr(),
                          ch._pair.data_ptr(), (nat.ctypes.c_uint64 * 2)(*nat.f64_mask([p])))
    ch.ring_p = nat.ctypes.pointer(ch.ring)
    ch._maps = {}
    return ch


@pytest.fixture(scope="module")
def c2_digests(golden_dir):
    with open(os.path.join(golden_dir, "c2_digests.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("L", [4, 12, 24])
def test_c2_full_size_digest(c2_digests, L):
    """One HMult and one HRot at the benchmark's full size (N=2^16, L limbs,
    dnum=3, k special primes) equal the oracle's outputs, compared through
    the SHA-256 of the coefficient planes the oracle produced on the CPU box
    (tests/golden/make_c2_digest.py), both through the batched engine the
    bench times (B=1 with a per-item key pointer) and the HE API."""
    g = c2_digests[f"L{L}"]
    n = g["n"]
    params, alpha, k = _c2_params(L, n)
    # the oracle's key stream (numpy sampler) and its HW-192 secret
    cust = he_api.keygen(params, {g["rot_step"]}, backend="ckks", rng_seed=g["key_seed"],
                         prime_layout="baseline", dnum=DNUM, secret_hw=g["secret_hw"],
                         sampler="numpy")
    be = cust.backend
    assert be.chain.all_primes == g["all_primes"]
    lvl = g["level"]
    rng = np.random.default_rng(g["plane_seed"])
    pa, pb = (_planes(be.chain.limbs_at(lvl), n, rng) for _ in range(2))
    assert [_sha(pa), _sha(pb)] == g["inputs_sha256"]
    a = be.payload_from_planes(pa, lvl).data
    b = be.payload_from_planes(pb, lvl).data
    hm = be.batch_hmult(a[None], b[None], lvl)[0]
    hr = be.batch_hrot(a[None], [g["rot_step"]], lvl)[0]
    assert _sha(be.planes_of(_wrap_payload(hm, lvl - 1))) == g["hmult_sha256"]
    assert _sha(be.planes_of(_wrap_payload(hr, lvl))) == g["hrot_sha256"]
    ev = cust.evaluator
    ca, cb = be._wrap(_wrap_payload(a, lvl), lvl, 0), be._wrap(_wrap_payload(b, lvl), lvl, 0)
    assert _sha(be.planes_of(ev.mul(ca, cb).payload)) == g["hmult_sha256"]
    assert _sha(be.planes_of(ev.rotate(ca, g["rot_step"]).payload)) == g["hrot_sha256"]


@pytest.mark.parametrize("case", ["c2_L24", "c2_L23_short_digit", "bootstrap_layout_low_p"])
def test_fused_ntt_mac_equals_unfused(case):
    """ckb_ks_ntt_mac (the digits' row-phase NTT fused with the key inner
    product, N=2^16) gives the same ciphertexts as the unfused transform +
    ckb_ks_inner, for batched HMult and per-item-key HRot: the config-2 chain,
    a short last digit (L=23, digits 8/8/7) and the bootstrap layout (60-bit Q
    primes: integer-class rows in the fused kernel) with a level-aware special
    modulus (keys over Q u P', k' < k)."""
    n = 1 << 16
    if case.startswith("c2"):
        L = 24 if case == "c2_L24" else 23
        params, _, _ = _c2_params(L, n)
        opts = dict(prime_layout="baseline", dnum=DNUM, secret_hw=192)
    else:
        from paper_2506_19693_b200.scheme import SchemeParams

        params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 4 + (60,) * 2 + (360,),
                              scale_bits=45, level=6, bootstrap_depth=2)
        opts = dict(prime_layout="bootstrap", dnum=3, secret_hw=64, low_special=[(4, 4)])
    rng = np.random.default_rng(3)
    steps = [int(s) for s in rng.choice(np.arange(1, n // 2), size=3, replace=False)]
    cust = he_api.keygen(params, set(steps), backend="ckks", rng_seed=5, **opts)
    be = cust.backend
    ch = be.chain
    for lvl in sorted({params.level, 3}):
        m = ch.level_limbs[lvl]
        x = torch.stack([be.payload_from_planes(_planes(ch.limbs_at(lvl), n, rng), lvl).data
                         for _ in range(3)])
        y = torch.stack([be.payload_from_planes(_planes(ch.limbs_at(lvl), n, rng), lvl).data
                         for _ in range(3)])
        outs = []
        for fused in (True, False):
            type(ch).fuse_ks_mac = fused
            try:
                outs.append((be.batch_hmult(x, y, lvl).clone(), be.batch_hrot(x, steps, lvl).clone(),
                             be._hrot(x, lvl, galois=be.galois_for_step[steps[0]],
                                      key=be.rotation_key(be.galois_for_step[steps[0]])).clone()))
            finally:
                type(ch).fuse_ks_mac = False
        for a, b in zip(*outs):
            assert torch.equal(a.view(torch.int64), b.view(torch.int64)), (case, lvl, m)
