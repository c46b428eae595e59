"""NTT-friendly prime chains (host side, runs once per parameter set).

Three layouts:

``reference``  — the reference's own chain (ckks/ntt.py:41-78, ckks/ring.py:24-53):
                 every limb below 2^31, wide entries split into several primes
                 nearest to an equal share, rescale entries chosen top-down so
                 the level scale schedule stays near nominal.  Identical primes
                 to the reference (checked in tests/test_host.py).
``baseline``   — BASELINE.json's rule: one prime per chain entry of <= 60 bits,
                 the largest prime = 1 mod 2N below 2^bits (wider entries become
                 ceil(bits/60) such primes).  Used for configs 1-2.
``bootstrap``  — for parameter sets with bootstrap_depth > 0: the user levels
                 1..refresh_level follow ``schedule`` at 2^scale_bits, the
                 bootstrapping levels above use the largest primes below
                 2^bits of their chain entries (~60 bits).  The level schedule
                 stays exact: above refresh_level scale_at[l] =
                 sqrt(scale_at[l-1] q_l), rising towards q (fresh encryptions at
                 the top are encoded at ~2^60); the bootstrapper itself tracks
                 scales explicitly (bootstrap.py).
``schedule``   — one prime per entry, rescale primes nearest to
                 scale_at[l]^2 / 2^scale_bits top-down (the reference's
                 schedule-stabilising rule with single word-size primes); keeps
                 deep chains (N=2^16, L=24) on a finite scale schedule.
"""

from __future__ import annotations

import math

import numpy as np

from .he_errors import InvalidParameters

REF_MAX_LIMB_BITS = 30
MAX_PRIME_BITS = 60  # every prime < 2^60: lazy [0, 8p) butterflies need p < 2^61, and the
                     # carry-free split dot products (modarith.cuh Acc4) need one operand < 2^60
_WITNESSES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (fixed witness set)."""
    if n < 2:
        return False
    for w in _WITNESSES:
        if n % w == 0:
            return n == w
    d, s = n - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    for a in _WITNESSES:
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def nearest_prime(target: int, two_n: int, used: set, max_bits: int) -> int:
    """Unused prime = 1 mod 2N closest to target (ties: the larger candidate
    first, the search order of ntt.py:43-52), below 2^(max_bits+1)."""
    k0 = max(1, round((target - 1) / two_n))
    limit = 1 << (max_bits + 1)
    for off in range(1 << 22):
        for k in (k0 + off, k0 - off):
            if k < 1:
                continue
            p = two_n * k + 1
            if p >= limit or p <= two_n or p in used:
                continue
            if is_prime(p):
                return p
    raise InvalidParameters(f"no NTT prime near {target} for 2N={two_n}")


def split_entry(target: float, two_n: int, used: set) -> list:
    """Reference split of one chain entry into sub-2^31 primes (ntt.py:56-73)."""
    bits = np.log2(target)
    if bits < 2:
        raise InvalidParameters(f"modulus entry of {bits:.1f} bits is too small")
    parts = 1
    while bits / parts > REF_MAX_LIMB_BITS:
        parts += 1
    remaining = float(target)
    out = []
    for i in range(parts):
        p = nearest_prime(round(remaining ** (1.0 / (parts - i))), two_n, used, REF_MAX_LIMB_BITS)
        used.add(p)
        out.append(p)
        remaining /= p
    return out


def largest_below(bits: int, two_n: int, used: set) -> int:
    if bits > MAX_PRIME_BITS:
        raise InvalidParameters(f"{bits}-bit primes exceed the {MAX_PRIME_BITS}-bit kernel limit")
    k = ((1 << bits) - 2) // two_n
    while k > 0:
        p = two_n * k + 1
        if p not in used and is_prime(p):
            return p
        k -= 1
    raise InvalidParameters(f"no {bits}-bit prime = 1 mod {two_n}")


def _wide(bits: int, two_n: int, used: set) -> list:
    parts = max(1, -(-bits // 60))
    out = []
    for _ in range(parts):
        p = largest_below(bits // parts, two_n, used)
        used.add(p)
        out.append(p)
    return out


def build_chain(params, layout: str = "reference"):
    """Returns (entry_primes, scale_at) with entry_primes ordered
    [base, level 1 .. level L, special] as ring.py:42-45."""
    n = params.poly_degree
    two_n = 2 * n
    chain = tuple(params.modulus_chain)
    level = params.level
    used: set = set()
    nominal = float(2 ** params.scale_bits)
    scale_at = [0.0] * (level + 1)
    scale_at[level] = nominal
    rescale = [None] * level
    if layout == "reference":
        base = split_entry(2.0 ** chain[0], two_n, used)
        special = split_entry(2.0 ** chain[-1], two_n, used)
        for lv in range(level, 0, -1):
            entry = split_entry(scale_at[lv] ** 2 / nominal, two_n, used)
            rescale[lv - 1] = entry
            scale_at[lv - 1] = scale_at[lv] ** 2 / math.prod(entry)
    elif layout == "bootstrap":
        base = _wide(chain[0], two_n, used)
        special = _wide(chain[-1], two_n, used)
        rl = params.refresh_level
        top_primes = {}
        for lv in range(level, rl, -1):
            p = largest_below(chain[lv], two_n, used)
            used.add(p)
            top_primes[lv] = p
        scale_at[rl] = nominal
        for lv in range(rl, 0, -1):
            p = nearest_prime(round(scale_at[lv] ** 2 / nominal), two_n, used, MAX_PRIME_BITS - 1)
            used.add(p)
            rescale[lv - 1] = [p]
            scale_at[lv - 1] = scale_at[lv] ** 2 / p
        for lv in range(rl + 1, level + 1):  # consistent upward: s_l = sqrt(s_{l-1} q_l)
            rescale[lv - 1] = [top_primes[lv]]
            scale_at[lv] = math.sqrt(scale_at[lv - 1] * top_primes[lv])
    elif layout in ("baseline", "schedule"):
        base = _wide(chain[0], two_n, used)
        special = _wide(chain[-1], two_n, used)
        for lv in range(level, 0, -1):
            if layout == "baseline":
                p = largest_below(chain[lv], two_n, used)
            else:
                p = nearest_prime(round(scale_at[lv] ** 2 / nominal), two_n, used, MAX_PRIME_BITS - 1)
            used.add(p)
            rescale[lv - 1] = [p]
            scale_at[lv - 1] = scale_at[lv] ** 2 / p
    else:
        raise InvalidParameters(f"unknown prime layout {layout!r}")
    return [base] + rescale + [special], scale_at
