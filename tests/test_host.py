"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side table builders and prime chains agree with the oracle/reference, the
HE-API mirror keeps the reference's bookkeeping rules, and the device modular
arithmetic is exact (compiled for the host with g++)."""

import os
import re
import shutil
import subprocess
import sys

import numpy as np
import pytest

from oracle import ckks_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    from paper_2506_19693_b200 import _native

    header = open(os.path.join(ROOT, "include", "ckks_b200.h")).read()
    declared = set(re.findall(r"\b(?:int|int64_t|uint64_t)\s+(ckb_\w+)\s*\(", header))
    assert declared == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(_native.LIB, name)
    assert _native.LIB.ckb_version() == 1


@pytest.mark.parametrize("logn,bits", [(4, 27), (10, 30), (12, 40), (16, 60)])
def test_build_tables_match_oracle_plan(logn, bits):
    from paper_2506_19693_b200 import _native

    n = 1 << logn
    p = O.largest_ntt_prime_below(bits, 2 * n, set())
    mods, ntt, pair = _native.build_tables(logn, [p])
    plan = O.NttPlan(p, n)
    t = ntt.reshape(1, 2, n, 2)
    if p < 2**46:  # FP64 NTT path, per direction: [N] double(w), then the same entries
        # with the two bottom stages' blocks interleaved by 16-byte chunk per warp
        # (ops.cu ckb_build_tables / ntt.cu load_tw_f64_perm)
        d = ntt.view(np.float64).reshape(1, 2, 2, n)
        assert [int(v) for v in d[0, 0, 0]] == [int(v) for v in plan.psi_brv]
        assert [int(v) for v in d[0, 1, 0]] == [int(v) for v in plan.inv_psi_brv]
        for dr, w in ((0, plan.psi_brv), (1, plan.inv_psi_brv)):
            want = [int(v) for v in w]
            if n >= 512:
                for nt, lo in ((8, n // 2), (4, n // 4)):
                    for b0 in range(lo, 2 * lo, 32 * nt):
                        for lane in range(32):
                            for e in range(nt):
                                want[b0 + (e // 2) * 64 + 2 * lane + (e & 1)] = int(
                                    w[b0 + nt * lane + e])
            assert [int(v) for v in d[0, dr, 1]] == want
    else:
        assert [int(v) for v in t[0, 0, :, 0]] == [int(v) for v in plan.psi_brv]
        assert [int(v) for v in t[0, 1, :, 0]] == [int(v) for v in plan.inv_psi_brv]
        assert [int(v) for v in t[0, 0, :8, 1]] == [(int(w) << 64) // p
                                                   for w in plan.psi_brv[:8]]
    assert int(mods[0, 0]) == p and int(mods[0, 4]) == pow(n, -1, p)
    assert int(mods[0, 6]) == int(plan.inv_psi_brv[1]) * pow(n, -1, p) % p


def test_build_tables_rejects_bad_primes():
    from paper_2506_19693_b200 import _native

    with pytest.raises(_native.NativeError):
        _native.build_tables(10, [12289 * 2**40 + 1])  # >= 2^62 or not = 1 mod 2N


def test_reference_layout_primes_match_reference(golden_dir):
    from paper_2506_19693_b200.primes import build_chain
    from paper_2506_19693_b200.scheme import SchemeParams

    g = np.load(os.path.join(golden_dir, "ref_ckks_n512.npz"))
    n, level, sb = (int(v) for v in g["params"])
    params = SchemeParams(poly_degree=n, modulus_chain=tuple(int(v) for v in g["chain"]),
                          scale_bits=sb, level=level)
    entries, scale_at = build_chain(params, "reference")
    allp = [p for e in entries for p in e]
    assert allp == [int(v) for v in g["all_primes"]]
    assert scale_at == [float(v) for v in g["scale_at"]]


@pytest.mark.parametrize("layout", ["reference", "baseline", "schedule"])
def test_layouts_match_oracle_chain(layout):
    from paper_2506_19693_b200.primes import build_chain
    from paper_2506_19693_b200.scheme import make_params

    params = make_params(level=8, scale_bits=40, poly_degree=4096)
    entries, scale_at = build_chain(params, layout)
    ch = O.Chain(4096, params.modulus_chain, 40, 8, layout)
    assert entries == ch.entry_primes
    assert scale_at == ch.scale_at


def test_config1_baseline_primes():
    # the 60-bit base and special primes for N=2^12
    from paper_2506_19693_b200.primes import build_chain
    from paper_2506_19693_b200.scheme import make_params

    entries, scale_at = build_chain(make_params(level=8, scale_bits=40, poly_degree=4096),
                                    "baseline")
    assert entries[0] == [1152921504606830593]
    assert entries[-1] == [1152921504606748673]
    assert all(len(e) == 1 and e[0] < 2**40 for e in entries[1:-1])
    assert all(abs(np.log2(s) - 40) < 0.01 for s in scale_at)


def test_modarith_exact_on_host():
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    exe = os.path.join("/tmp", f"ckb_modarith_{os.getpid()}")
    src = os.path.join(ROOT, "tests", "native", "test_modarith.cpp")
    subprocess.run([gxx, "-O2", "-std=c++17", "-o", exe, src], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fails=0" in r.stdout


# ---------------------------------------------------------------------------
# HE API mirror: the reference contract rules on a float payload stand-in
# ---------------------------------------------------------------------------


class _FloatBackend:
    """Minimal payload hooks (plain float arrays) to exercise the shared
    bookkeeping of he_api.Backend; the B200 backend inherits exactly this."""

    backend_id = "float"

    def _payload_elementwise(self, kind, a, b, out_level):
        x = a.payload
        y = b.payload if kind.endswith("_ct") else b.values
        return {"add": x + y, "sub": x - y, "mul": x * y}[kind[:3]]

    def _payload_rotate(self, a, k):
        return np.roll(a.payload, -k)

    def _payload_encrypt(self, pv, level, serial):
        return pv.values.copy()

    def _payload_decrypt(self, cv):
        return cv.payload

    def _payload_bootstrap(self, cv, serial):
        return cv.payload.copy()


def _float_custodian(level=3, rots=(1, -1)):
    from paper_2506_19693_b200 import he_api
    from paper_2506_19693_b200.scheme import make_params

    params = make_params(level=level, scale_bits=40, poly_degree=16, bootstrap_depth=1)
    cls = type("FB", (_FloatBackend, he_api.Backend), {})
    return he_api.KeyCustodian(cls(params, "ks"), rots)


def test_he_api_levels_depth_and_errors():
    from paper_2506_19693_b200 import he_api, he_errors

    cust = _float_custodian()
    ev = cust.evaluator
    v = np.arange(8, dtype=np.float64)
    a = cust.encrypt(ev.plain(v))
    b = cust.encrypt(ev.plain(v))
    with cust.ledger.iteration():
        m = ev.mul(a, b)
        assert (m.level_remaining, m.depth) == (2, 1)
        s = ev.add(m, a)
        assert (s.level_remaining, s.depth) == (2, 1)
        m2 = ev.mul(s, ev.plain(v))
        assert (m2.level_remaining, m2.depth) == (1, 2)
        r = ev.rotate(m2, -1)
        assert np.array_equal(cust.decrypt(r).values, np.roll(v * v * v + v * v, 1))
    assert cust.ledger.iteration_depths == [2]
    x = a
    for _ in range(3):
        x = ev.mul(x, a)
    with pytest.raises(he_errors.LevelExhausted):
        ev.mul(x, a)
    with pytest.raises(he_errors.MissingRotationKey):
        ev.rotate(a, 2)
    with pytest.raises(he_errors.IncompatibleOperands):
        ev.add(a, he_api.make_plain(v, 4, 40.0))
    other = _float_custodian()
    other.backend.keyset_id = "other"
    with pytest.raises(he_errors.IncompatibleOperands):
        ev.add(a, other.encrypt(ev.plain(v)))
    bs = cust.bootstrap(x)
    assert bs.level_remaining == 2 and bs.depth == 0 and cust.ledger.bootstrap_count == 1
    with pytest.raises(he_errors.IncompatibleOperands):
        he_api.make_plain(np.zeros(9), 8, 40.0)


def test_scheme_params_rules():
    from paper_2506_19693_b200.he_errors import InvalidParameters, SecurityError
    from paper_2506_19693_b200.scheme import SchemeParams, make_params

    with pytest.raises(SecurityError):
        make_params(level=10, scale_bits=40, poly_degree=2**12, security_claim=128)
    ok = make_params(level=24, scale_bits=49, poly_degree=2**16, bootstrap_depth=16,
                     security_claim=128)
    assert ok.refresh_level == 8 and ok.slot_count == 2**15
    with pytest.raises(InvalidParameters):
        SchemeParams(poly_degree=1000, modulus_chain=(60, 60, 60), scale_bits=40, level=1)
    with pytest.raises(InvalidParameters):
        SchemeParams(poly_degree=1024, modulus_chain=(60, 60), scale_bits=40, level=1)


# ---------------------------------------------------------------------------
# Drop-in registration into the real reference (build container only)
# ---------------------------------------------------------------------------

REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_plugin_swaps_reference_backend_class():
    sys.path.insert(0, REF_SRC)
    try:
        import ciphermlp.ckks.backend as rb
        from ciphermlp.api import keygen as ref_keygen
        from ciphermlp.params import make_params as ref_make_params

        from paper_2506_19693_b200 import plugin

        cls, old = plugin.install(prime_layout="reference")
        try:
            assert rb.CkksBackend is cls and cls.backend_id == "ckks"
            import ciphermlp.api as rapi
            import ciphermlp.errors as rerr

            assert issubclass(cls, rapi.Backend) and cls._errors is rerr
            params = ref_make_params(level=2, scale_bits=40, poly_degree=1024)
            import torch

            if not torch.cuda.is_available():
                with pytest.raises(RuntimeError, match="CUDA"):
                    ref_keygen(params, {1}, backend="ckks", rng_seed=0)
        finally:
            plugin.uninstall(old)
        assert rb.CkksBackend is old
    finally:
        sys.path.remove(REF_SRC)
