"""Out-of-bounds write guard (compute-sanitizer is closed on this GPU pool: its
runs left GPUs needing a reset).  Every kernel wrapper that takes an output
tensor writes into a view carved out of a larger buffer whose head and tail
are filled with a canary pattern; after the call the canaries must be
untouched and the result must equal the same call into a plain tensor.  Run
at the benchmark's shapes (N=2^16, L=24, alpha=8, k=6, two-phase NTTs) and at
N=2^10 (single-phase NTTs), every kernel family of the key-switching path."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_19693_b200 import he_api  # noqa: E402
from paper_2506_19693_b200.scheme import make_params  # noqa: E402

CANARY = 0x5AA5C33C0FF0E11E
PAD = 4096 + 8  # words on each side (more than a 16-byte vector / tile overrun)


def guarded(*shape):
    numel = int(np.prod(shape))
    big = torch.full((2 * PAD + numel,), CANARY, dtype=torch.int64, device="cuda")
    return big, big[PAD:PAD + numel].view(*shape).view(torch.uint64)


def intact(big):
    head, tail = big[:PAD], big[-PAD:]
    return bool((head == CANARY).all()) and bool((tail == CANARY).all())


@pytest.mark.parametrize("n,L", [(1 << 16, 24), (1 << 10, 24), (1 << 10, 4)])
def test_kernels_write_only_their_outputs(n, L):
    alpha = -(-L // 3)
    k = -(-40 * alpha // 60)
    params = make_params(level=L - 1, scale_bits=40, poly_degree=n, first_bits=40,
                         special_bits=60 * k)
    cust = he_api.keygen(params, {1, 3}, backend="ckks", rng_seed=4, prime_layout="baseline",
                         dnum=3, secret_hw=64)
    be = cust.backend
    ch = be.chain
    lvl = params.level
    m = ch.level_limbs[lvl]
    B = 2
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)

    def rand(*lead):
        t = torch.empty(*lead, m, n, dtype=torch.int64, device="cuda")
        for i, p in enumerate(ch.limbs_at(lvl)):
            t[..., i, :].random_(0, p, generator=gen)
        return t.view(torch.uint64)

    a, b = rand(B, 2), rand(B, 2)
    checks = []

    def check(name, fn, shape, ref=None):
        big, out = guarded(*shape)
        r = fn(out)
        torch.cuda.synchronize()
        assert intact(big), f"{name} wrote outside its output"
        if ref is not None:
            assert torch.equal(out.view(torch.int64), ref.view(torch.int64)), name
        checks.append(name)
        return r

    # NTT in place and out of place (rows of the whole batch)
    big, x = guarded(B, 2, m, n)
    x.copy_(a)
    ch.ntt_fwd(x, m)
    ch.ntt_inv(x, m)
    torch.cuda.synchronize()
    assert intact(big) and torch.equal(x.view(torch.int64), a.view(torch.int64))
    check("ntt_from", lambda o: ch.ntt_from(a[:, 1], B, m, 2 * m * n, inverse=True, out=o),
          (B, m, n))
    check("tensor", lambda o: ch.tensor(a, b, m, out=o), (B, 3, m, n))
    check("elementwise", lambda o: ch.mul(a, b, m, out=o), (B, 2, m, n), ch.mul(a, b, m))
    check("automorphism_ntt", lambda o: ch.automorphism_ntt(a, 25, out=o), (B, 2, m, n))
    d2 = ch.ntt_from(a[:, 1], B, m, 2 * m * n, inverse=True)
    rows = len(ch.digit_basis(m, be.alpha, True))
    digits = check("modup", lambda o: ch.modup(d2, m, be.alpha, be._bconv(m), batch=B,
                                                skip_own=True, out=o), (B, rows, n))
    basis = ch.digit_basis(m, be.alpha, True)
    ref_digits = digits.clone()
    ch.ntt_fwd(ref_digits, len(basis), ch.cmap(basis))
    ext = m + ch.k
    acc = check("ks_inner", lambda o: ch.ks_inner(ref_digits, m, be.alpha,
                                                  key=be.relin_key.data, own=a[:, 1],
                                                  own_bstride=2 * m * n, out=o), (B, 2, ext, n))
    if n >= 1 << 16:
        bigd, dg = guarded(B, rows, n)
        dg.copy_(digits)
        check("ks_ntt_mac", lambda o: ch.ks_ntt_mac(dg, m, be.alpha, key=be.relin_key.data,
                                                    own=a[:, 1], own_bstride=2 * m * n, out=o),
              (B, 2, ext, n), acc)
        assert intact(bigd), "ks_ntt_mac wrote outside its digits scratch"
    check("divround_ntt", lambda o: ch.divround_ntt(acc.view(2 * B, ext, n), 2 * B, ext, ch.k,
                                                    1, addend=a, addend_polys=2,
                                                    addend_period=2, addend_stride=2,
                                                    addend_tail=a[:, :, m - 1:m].reshape(
                                                        2 * B, 1, n).contiguous(),
                                                    basis=ch.ext_basis(m), out=o),
          (2 * B, m - 1, n))
    coeffs = torch.randint(-(1 << 40), 1 << 40, (B, n), dtype=torch.int64, device="cuda")
    check("from_i64", lambda o: ch.from_i64(coeffs, m, out=o), (B, m, n))
    assert len(checks) >= 8
