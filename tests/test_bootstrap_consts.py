"""Bootstrapping constants (paper_2506_19693_b200/bootstrap_consts.py) against
direct numpy evaluation — the f64 restatement check of SURVEY.md H5 (≤ 1e-6;
we require ≤ 1e-9)."""

import numpy as np
import pytest

from paper_2506_19693_b200 import bootstrap_consts as B


@pytest.mark.parametrize("logn", [4, 6, 10])
def test_special_fft_is_the_slot_map(logn):
    n = 1 << logn            # ring degree
    slots = n // 2
    rng = np.random.default_rng(logn)
    c = rng.integers(-1000, 1000, n).astype(np.float64)
    cp = c[:slots] + 1j * c[slots:]
    z = B.special_fft(cp, 2 * n)
    zeta = np.exp(1j * np.pi / n)
    rg = B.rot_group(slots, 2 * n)
    direct = np.array([np.sum(c * zeta ** (rg[k] * np.arange(n))) for k in range(slots)])
    assert np.max(np.abs(z - direct)) <= 1e-9 * np.max(np.abs(direct))


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_grouped_transforms_invert(levels):
    n = 1 << 9
    slots = n // 2
    rng = np.random.default_rng(levels)
    cp = rng.normal(size=slots) + 1j * rng.normal(size=slots)
    z = B.special_fft(cp, 2 * n)
    cts = B.grouped_transform(slots, 2 * n, levels, inverse=True)
    x = z.copy()
    for m in cts:
        x = B.apply_diagonals(m, x)
    x /= slots
    bits = slots.bit_length() - 1
    idx = np.arange(slots)
    rev = np.zeros_like(idx)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    assert np.max(np.abs(x - cp[rev])) <= 1e-9          # CtS = P V^-1
    stc = B.grouped_transform(slots, 2 * n, levels, inverse=False)
    y = x.copy()
    for m in stc:
        y = B.apply_diagonals(m, y)
    assert np.max(np.abs(y - z)) <= 1e-9 * np.max(np.abs(z))   # StC = V P


def test_bsgs_matches_direct():
    n = 1 << 10
    slots = n // 2
    rng = np.random.default_rng(0)
    x = rng.normal(size=slots) + 1j * rng.normal(size=slots)
    for m in B.grouped_transform(slots, 2 * n, 3, inverse=True):
        plan = B.bsgs_plan(m, slots)
        assert np.max(np.abs(B.bsgs_apply(plan, x) - B.apply_diagonals(m, x))) <= 1e-9
        assert len(B.bsgs_rotations(plan, slots)) <= 16


def test_evalmod_chebyshev_accuracy():
    K, r = 28, 2
    f = B.evalmod_function(K, r)
    c = B.cheb_coeffs(f, 119)
    xs = np.linspace(-1, 1, 20001)
    err = np.max(np.abs(np.polynomial.chebyshev.chebval(xs, c) - f(xs)))
    assert err <= 1e-9
    # r double angles give sin(2π(K+1)x)
    y = f(xs)
    for _ in range(r):
        y = 2 * y * y - 1
    assert np.max(np.abs(y - np.sin(2 * np.pi * (K + 1) * xs))) <= 1e-9
