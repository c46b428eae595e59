"""Tensor-core basis conversions (csrc/tc.cu, tcgen05.mma kind::i8).

ModUp (keys.py:84-90) and the fast-conversion ModDown correction
(keys.py:98-99 + ring.py:165-189) run as byte-sliced u8 GEMMs on the tensor
cores when the chain sets CKB_RING_TC (the default).  These tests pin:
  * the operand layout / descriptors: one tcgen05 tile against numpy;
  * bit-identity with the CUDA-core kernels (CKB_RING_TC cleared) on every
    key-switch path of the benchmark and the training configs: batched HMult
    (ModDown + fused rescale), per-item-key HRot, a single-key rotation, ModUp
    without skip_own, a short last digit, 60-bit Q primes with a level-aware
    special modulus (8-column outputs), the forced exact-rho path, and the
    reference prime layout (sub-2^31 primes: the small-prime reduction).
The oracle comparisons of the same paths (tests/test_gpu_headline.py,
test_gpu_parity.py) run with the tensor cores on."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2506_19693_b200 import _native as nat  # noqa: E402
from paper_2506_19693_b200 import he_api  # noqa: E402
from paper_2506_19693_b200.scheme import SchemeParams, make_params  # noqa: E402


@pytest.mark.parametrize("k,n", [(32, 16), (64, 128), (96, 176), (128, 256), (256, 64)])
def test_tc_selftest_gemm(k, n):
    rng = np.random.default_rng(k * 1000 + n)
    a = rng.integers(0, 256, (128, k), dtype=np.uint8)
    b = rng.integers(0, 256, (n, k), dtype=np.uint8)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    d = torch.empty(128, n, dtype=torch.int32, device="cuda")
    nat.check(nat.LIB.ckb_tc_selftest(nat.ptr(ta), nat.ptr(tb), nat.ptr(d), k, n,
                                      nat.stream_handle()), "tc_selftest")
    want = a.astype(np.int64) @ b.astype(np.int64).T
    assert np.array_equal(d.cpu().numpy().astype(np.int64), want)


def _planes(primes, n, rng):
    return np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
                     for _ in range(2)])


def _case(case, n):
    if case.startswith("c2"):
        L = {"c2_L24": 24, "c2_L12": 12, "c2_L4": 4, "c2_L23_short": 23}[case]
        alpha = -(-L // 3)
        k = -(-40 * alpha // 60)
        params = make_params(level=L - 1, scale_bits=40, poly_degree=n, first_bits=40,
                             special_bits=60 * k)
        return params, dict(prime_layout="baseline", dnum=3, secret_hw=192)
    if case == "boot_low_p":
        params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 4 + (60,) * 2 + (360,),
                              scale_bits=45, level=6, bootstrap_depth=2)
        return params, dict(prime_layout="bootstrap", dnum=3, secret_hw=64,
                            low_special=[(4, 4)])
    if case == "c3_layout":  # config-3 chain: 45-bit (6 columns) and 60-bit (8) outputs,
        # 256- and 512-column accumulators (2 and 1 CTAs per SM, 8 / 16 warps each)
        params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,),
                              scale_bits=45, level=24, bootstrap_depth=16)
        return params, dict(prime_layout="bootstrap", dnum=3, secret_hw=64)
    if case == "reference_layout":  # config-1 style chain: sub-2^31 primes, per-limb digits
        params = make_params(level=3, scale_bits=26, poly_degree=n, first_bits=40,
                             special_bits=200)
        return params, dict(prime_layout="reference", secret_hw=64)
    raise ValueError(case)


def _outputs(be, x, y, steps, lvl):
    ch = be.chain
    m = ch.level_limbs[lvl]
    coeff = x[:, 0].contiguous()  # any canonical residues will do for ModUp
    # ModUp's own outputs canonical (the lazy [0, 3p) form only feeds NTTs)
    lazy = ch.set_ring_flag(nat.RING_LAZY_BCONV, False)
    try:
        mu = ch.modup(coeff, m, be.alpha, be._bconv(m, ch.k), skip_own=False).clone()
    finally:
        ch.set_ring_flag(nat.RING_LAZY_BCONV, lazy)
    return (be.batch_hmult(x, y, lvl).clone(), be.batch_hrot(x, steps, lvl).clone(),
            be._hrot(x, lvl, galois=be.galois_for_step[steps[0]],
                     key=be.rotation_key(be.galois_for_step[steps[0]])).clone(), mu)


@pytest.mark.parametrize("case", ["c2_L24", "c2_L12", "c2_L4", "c2_L23_short", "boot_low_p",
                                  "c3_layout", "reference_layout", "c2_L24_hps_exact"])
def test_tc_bit_identical_to_cuda_cores(case):
    n = 4096
    exact = case.endswith("_hps_exact")
    params, opts = _case(case.replace("_hps_exact", ""), n)
    rng = np.random.default_rng(11)
    steps = [int(s) for s in rng.choice(np.arange(1, n // 2), size=3, replace=False)]
    cust = he_api.keygen(params, set(steps), backend="ckks", rng_seed=5, **opts)
    be = cust.backend
    ch = be.chain
    if exact:
        ch.set_ring_flag(nat.RING_HPS_EXACT, True)
    try:
        for lvl in sorted({params.level, max(1, params.level // 2)}):
            x = torch.stack([be.payload_from_planes(_planes(ch.limbs_at(lvl), n, rng), lvl).data
                             for _ in range(3)])
            y = torch.stack([be.payload_from_planes(_planes(ch.limbs_at(lvl), n, rng), lvl).data
                             for _ in range(3)])
            outs = []
            for tc in (True, False):
                prev = ch.set_ring_flag(nat.RING_TC, tc)
                try:
                    outs.append(_outputs(be, x, y, steps, lvl))
                finally:
                    ch.set_ring_flag(nat.RING_TC, prev)
            for i, (a, b) in enumerate(zip(*outs)):
                assert torch.equal(a.view(torch.int64), b.view(torch.int64)), (case, lvl, i)
    finally:
        ch.set_ring_flag(nat.RING_HPS_EXACT, False)


def test_tc_lazy_outputs_reduce_to_the_canonical_ones():
    """CKB_RING_LAZY_BCONV: ModUp outputs in [0, 3p), congruent to the canonical ones."""
    params, opts = _case("c2_L24", 4096)
    cust = he_api.keygen(params, set(), backend="ckks", rng_seed=2, **opts)
    be = cust.backend
    ch = be.chain
    lvl = params.level
    m = ch.level_limbs[lvl]
    rng = np.random.default_rng(4)
    x = torch.stack([be.payload_from_planes(_planes(ch.limbs_at(lvl), 4096, rng), lvl).data
                     for _ in range(2)])[:, 0].contiguous()
    outs = {}
    for lazy in (True, False):
        prev = ch.set_ring_flag(nat.RING_LAZY_BCONV, lazy)
        outs[lazy] = ch.modup(x, m, be.alpha, be._bconv(m, ch.k), skip_own=False).cpu().numpy()
        ch.set_ring_flag(nat.RING_LAZY_BCONV, prev)
    ext = list(range(m)) + list(range(ch.lq, ch.lq + ch.k))
    nd = -(-m // be.alpha)
    primes = np.array([ch.all_primes[i] for i in ext], dtype=np.uint64)
    lz = outs[True].reshape(2, nd, len(ext), -1)
    cn = outs[False].reshape(2, nd, len(ext), -1)
    p = primes[None, None, :, None]
    assert np.all(lz < 3 * p) and np.array_equal(lz % p, cn) and np.all(cn < p)
    assert not np.array_equal(lz, cn)  # the lazy form is in use


def test_tc_default_on():
    """GpuChain turns the tensor-core path on unless CKB_NO_TC=1."""
    params, opts = _case("c2_L4", 1024)
    cust = he_api.keygen(params, set(), backend="ckks", rng_seed=1, **opts)
    ch = cust.backend.chain
    assert bool(ch.ring.flags & nat.RING_TC) == (os.environ.get("CKB_NO_TC") != "1")
    assert (ch.ring.wide_mask[0], ch.ring.wide_mask[1]) == nat.wide_mask(ch.all_primes)
    assert (ch.ring.mid_mask[0], ch.ring.mid_mask[1]) == nat.mid_mask(ch.all_primes)
