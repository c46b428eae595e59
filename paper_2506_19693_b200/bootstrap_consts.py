"""Host-side constants for CKKS bootstrapping.

The reference has no bootstrapping (its refresh decrypts and re-encrypts,
ckks/backend.py:195-206), so these follow the published algorithm the paper
cites (CoeffToSlot / EvalMod / SlotToCoeff) and are checked
against direct numpy evaluation in tests/test_bootstrap_consts.py (≤ 1e-9).

Slot convention (ckks/encoding.py:20-32): slot k of a plaintext m(X) is
m(ζ^{5^k}), ζ = e^{iπ/N}.  Writing the N real coefficients as N/2 complex
values c'_j = c_j + i c_{j+N/2}, the slots are z = V c' with
V_{kj} = ζ^{5^k j} (because ζ^{5^k N/2} = i).  V factors into a bit-reversal P
and log2(N/2) sparse butterfly stages ("special FFT"):

    V = B_{n} ... B_4 B_2 P,     B_len: (u, v) -> (u + ω v, u - ω v)
    ω = ζ^{(5^j mod 4len) * (2N / 4len)} for butterfly j of each block of len.

CoeffToSlot applies P V^{-1} = (1/n) I_2 ... I_n (I_len = 2 B_len^{-1});
SlotToCoeff applies V P = B_n ... B_2.  The bit-reversed slot order in
between is harmless because EvalMod is slot-wise.  Stages are grouped into
`levels` dense-diagonal matrices (products of consecutive stages), each
evaluated with baby-step/giant-step rotations.
"""

from __future__ import annotations

import math

import numpy as np


def rot_group(slots: int, two_n: int) -> np.ndarray:
    out = np.empty(slots, dtype=np.int64)
    e = 1
    for i in range(slots):
        out[i] = e
        e = e * 5 % two_n
    return out


def _omega(j, length, two_n, rg):
    lenq = 4 * length
    gap = two_n // lenq
    return np.exp(2j * np.pi * ((rg[j] % lenq) * gap) / two_n)


def stage_diagonals(slots: int, length: int, two_n: int, inverse: bool = False) -> dict:
    """Diagonals {offset: vector} of one butterfly stage with block size `length`
    ((M x)[p] = sum_k d_k[p] x[(p + k) mod slots]).  inverse=True gives
    I_len = 2 B_len^{-1}: (a, b) -> (a + b, (a - b) conj(ω))."""
    h = length // 2
    rg = rot_group(slots, two_n)
    d0 = np.zeros(slots, dtype=np.complex128)
    dp = np.zeros(slots, dtype=np.complex128)
    dm = np.zeros(slots, dtype=np.complex128)
    w = _omega(np.arange(h), length, two_n, rg)
    for i in range(0, slots, length):
        top = np.arange(i, i + h)
        bot = top + h
        if not inverse:
            d0[top] = 1.0
            dp[top] = w
            dm[bot] = 1.0
            d0[bot] = -w
        else:
            wc = np.conj(w)
            d0[top] = 1.0
            dp[top] = 1.0
            dm[bot] = wc
            d0[bot] = -wc
    out = {0: d0}
    out[h % slots] = out.get(h % slots, 0) + dp
    out[(-h) % slots] = out.get((-h) % slots, 0) + dm
    return out


def compose(a: dict, b: dict, slots: int) -> dict:
    """Diagonals of A·B (B applied first)."""
    out: dict = {}
    for k, ak in a.items():
        for l, bl in b.items():
            key = (k + l) % slots
            v = ak * np.roll(bl, -k)
            out[key] = out.get(key, 0) + v
    return {k: v for k, v in out.items() if np.any(v != 0)}


def apply_diagonals(diags: dict, x: np.ndarray) -> np.ndarray:
    out = np.zeros_like(x, dtype=np.complex128)
    for k, d in diags.items():
        out += d * np.roll(x, -k)
    return out


def special_fft(cp: np.ndarray, two_n: int) -> np.ndarray:
    """V c' via the stage factorisation (reference implementation for tests)."""
    n = cp.shape[0]
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros_like(idx)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    x = cp[rev].astype(np.complex128)
    length = 2
    while length <= n:
        x = apply_diagonals(stage_diagonals(n, length, two_n), x)
        length *= 2
    return x


def grouped_transform(slots: int, two_n: int, levels: int, inverse: bool) -> list:
    """Per-level diagonal dicts, in application order.

    inverse=False (SlotToCoeff, V P): stages len = 2, 4, ..., n.
    inverse=True (CoeffToSlot, P V^-1 without the 1/n): stages len = n, ..., 2
    of I_len."""
    logn = slots.bit_length() - 1
    lens = [1 << (s + 1) for s in range(logn)]
    if inverse:
        lens = lens[::-1]
    per = -(-logn // levels)
    groups = [lens[i:i + per] for i in range(0, logn, per)]
    mats = []
    for g in groups:
        m = None
        for length in g:
            st = stage_diagonals(slots, length, two_n, inverse)
            m = st if m is None else compose(st, m, slots)
        mats.append(m)
    return mats


def bsgs_plan(diags: dict, slots: int, n1: int = None):
    """Split offsets k*s (s = gcd stride) as (g*n1 + b)*s.  Returns
    (stride, n1, {g: {b: pre-rotated diagonal}}) with the giant-step
    pre-rotation folded in: pt_{g,b} = roll(d_{(g n1 + b) s}, g n1 s)."""
    offs = sorted(diags)
    nz = [o for o in offs if o]
    s = 0
    for o in nz:
        s = math.gcd(s, o)
    s = s or slots
    ks = []
    for o in offs:
        k = o // s
        if k > (slots // s) // 2:
            k -= slots // s
        ks.append((k, o))
    span = max(abs(k) for k, _ in ks) * 2 + 1
    if n1 is None:
        n1 = 1 << max(0, math.ceil(math.log2(math.sqrt(span))))
    plan: dict = {}
    for k, o in ks:
        g, b = divmod(k, n1)
        plan.setdefault(g, {})[b] = np.roll(diags[o], (g * n1 * s) % slots)
    return s, n1, plan


def bsgs_apply(plan_tuple, x: np.ndarray) -> np.ndarray:
    """Reference BSGS evaluation (numpy): sum_g rot(sum_b pt_gb * rot(x, b s), g n1 s)."""
    s, n1, plan = plan_tuple
    out = np.zeros_like(x, dtype=np.complex128)
    for g, row in plan.items():
        inner = np.zeros_like(out)
        for b, pt in row.items():
            inner += pt * np.roll(x, -b * s)
        out += np.roll(inner, -g * n1 * s)
    return out


def bsgs_rotations(plan_tuple, slots: int) -> set:
    s, n1, plan = plan_tuple
    rots = set()
    for g, row in plan.items():
        if g:
            rots.add((g * n1 * s) % slots)
        for b in row:
            if b:
                rots.add((b * s) % slots)
    return rots


def cheb_coeffs(fn, degree: int) -> np.ndarray:
    """Chebyshev interpolant of fn on [-1, 1] (first-kind basis)."""
    return np.polynomial.chebyshev.chebinterpolate(fn, degree)


def evalmod_function(K: int, r: int):
    """cos(2π((K+1)x - 1/4) / 2^r): r double-angle steps then give
    sin(2π (K+1) x), i.e. sin(2π u) for u = (K+1) x."""
    return lambda x: np.cos(2 * np.pi * ((K + 1) * np.asarray(x) - 0.25) / (1 << r))
