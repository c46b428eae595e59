"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference RNS-CKKS backend
(/root/reference/pkg/src/ciphermlp/ckks/{ntt,ring,keys,encoding,backend}.py),
used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
checker and the CPU timing baseline.  Nothing under paper_2506_19693_b200/ may
import it.

Two prime layouts are supported:
  * layout="reference" — the reference's own chain (ring.py:24-53): every limb
    below 2^31, entries split into several primes (mode A).  With this layout
    the oracle reproduces the reference bit for bit; that is pinned by
    tests/golden/ref_*.npz (generated from the real reference by
    tests/golden/make_golden.py) in tests/test_oracle_golden.py.
  * layout="baseline" / "schedule" — single 40/60-bit primes (BASELINE.json
    configs; mode B).  numpy uint64 would overflow, so limbs whose prime is
    >= 2^31 are held as dtype=object arrays of Python ints (exact, slow: small
    sizes only).  Hybrid key switching with digit size alpha > 1 follows the
    standard fast basis conversion; alpha == 1 is the reference's per-limb
    centered digit (keys.py:84-97).

Every function cites the reference line it restates.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

ERROR_SIGMA = 3.2  # keys.py:26
MAX_REF_LIMB_BITS = 30  # ntt.py:14
MAX_SAFE_COEFF = float(2**52)  # encoding.py:14


class OracleError(Exception):
    pass


class EncodingOverflowError(OracleError):
    pass


# ---------------------------------------------------------------------------
# primes (ntt.py:17-89)
# ---------------------------------------------------------------------------

_SMALL = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin (ntt.py:17-38)."""
    if n < 2:
        return False
    for p in _SMALL:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _SMALL:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def nearest_ntt_prime(target: int, two_n: int, used: set, max_bits: int = MAX_REF_LIMB_BITS) -> int:
    """Closest unused prime = 1 mod 2N below 2^(max_bits+1) (ntt.py:41-53)."""
    base = max(1, round((target - 1) / two_n))
    for offset in range(0, 1 << 22):
        for k in (base + offset, base - offset):
            if k < 1:
                continue
            p = two_n * k + 1
            if p >= 1 << (max_bits + 1) or p <= two_n:
                continue
            if p not in used and is_prime(p):
                return p
    raise OracleError(f"no NTT prime near {target}")


def primes_for_product(target: float, two_n: int, used: set) -> list:
    """Reference entry split (ntt.py:56-73)."""
    bits = np.log2(target)
    if bits < 2:
        raise OracleError("entry too small")
    n_limbs = 1
    while bits / n_limbs > MAX_REF_LIMB_BITS:
        n_limbs += 1
    remaining = float(target)
    out = []
    for i in range(n_limbs):
        share = remaining ** (1.0 / (n_limbs - i))
        p = nearest_ntt_prime(round(share), two_n, used)
        used.add(p)
        out.append(p)
        remaining /= p
    return out


def largest_ntt_prime_below(bits: int, two_n: int, used: set) -> int:
    """BASELINE rule: largest prime = 1 mod 2N below 2^bits, not yet used."""
    k = ((1 << bits) - 2) // two_n
    while k > 0:
        p = two_n * k + 1
        if p not in used and is_prime(p):
            return p
        k -= 1
    raise OracleError(f"no {bits}-bit NTT prime")


def primitive_2n_root(p: int, two_n: int) -> int:
    """ntt.py:81-89."""
    n = two_n // 2
    cof = (p - 1) // two_n
    for g in range(2, 10_000):
        psi = pow(g, cof, p)
        if psi != 1 and pow(psi, n, p) == p - 1:
            return psi
    raise OracleError("no primitive root")


def bit_reverse_perm(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros_like(idx)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev


def _dtype_for(p: int):
    return np.uint64 if p < (1 << 31) else object


def as_limb(values, p: int) -> np.ndarray:
    arr = np.asarray(values)
    if _dtype_for(p) is object:
        return np.array([int(v) for v in arr.tolist()], dtype=object)
    return arr.astype(np.uint64)


class NttPlan:
    """ntt.py:100-154 restated; works for any p < 2^62 via object arrays."""

    def __init__(self, p: int, n: int):
        self.p, self.n = p, n
        psi = primitive_2n_root(p, 2 * n)
        psi_inv = pow(psi, -1, p)
        pw, ipw = [], []
        a = b = 1
        for _ in range(n):
            pw.append(a)
            ipw.append(b)
            a = a * psi % p
            b = b * psi_inv % p
        rev = bit_reverse_perm(n)
        dt = _dtype_for(p)
        self.psi_brv = np.array(pw, dtype=object)[rev]
        self.inv_psi_brv = np.array(ipw, dtype=object)[rev]
        if dt is not object:
            self.psi_brv = self.psi_brv.astype(np.uint64)
            self.inv_psi_brv = self.inv_psi_brv.astype(np.uint64)
        self.n_inv = pow(n, -1, p)
        self._P = np.uint64(p) if dt is not object else p
        self._ninv = np.uint64(self.n_inv) if dt is not object else self.n_inv

    def forward(self, a: np.ndarray) -> np.ndarray:
        p = self._P
        x = as_limb(a, self.p).copy()
        n = self.n
        t, m = n, 1
        while m < n:
            t //= 2
            view = x.reshape(m, 2 * t)
            s = self.psi_brv[m:2 * m].reshape(m, 1)
            u = view[:, :t].copy()
            v = view[:, t:] * s % p
            view[:, t:] = (u + (p - v)) % p
            view[:, :t] = (u + v) % p
            m *= 2
        return x

    def inverse(self, a: np.ndarray) -> np.ndarray:
        p = self._P
        x = as_limb(a, self.p).copy()
        n = self.n
        t, m = 1, n
        while m > 1:
            h = m // 2
            view = x.reshape(h, 2 * t)
            s = self.inv_psi_brv[h:2 * h].reshape(h, 1)
            u = view[:, :t].copy()
            v = view[:, t:].copy()
            view[:, :t] = (u + v) % p
            view[:, t:] = (u + (p - v)) % p * s % p
            t *= 2
            m = h
        return x * self._ninv % p


def schoolbook_negacyclic(a, b, p: int) -> list:
    """ntt.py:157-169 (O(N^2) known-answer oracle)."""
    n = len(a)
    out = [0] * n
    for i, ai in enumerate(a):
        for j, bj in enumerate(b):
            k = i + j
            term = int(ai) * int(bj)
            if k < n:
                out[k] = (out[k] + term) % p
            else:
                out[k - n] = (out[k - n] - term) % p
    return [v % p for v in out]


# ---------------------------------------------------------------------------
# chain (ring.py:21-59)
# ---------------------------------------------------------------------------


class Chain:
    """Prime chain ordered [base | rescale entries 1..L | special].

    layout:
      "reference" — ring.py:24-45 exactly (entries split below 2^31);
      "baseline"  — one prime per <=60-bit entry, each the largest prime = 1 mod 2N
                    below 2^bits (BASELINE configs); an entry wider than 60 bits
                    becomes ceil(bits/60) equal primes;
      "schedule"  — one prime per entry, rescale primes picked top-down nearest to
                    scale_at[l]^2/nominal as ring.py:33-41 does (keeps deep chains
                    stable).
    """

    def __init__(self, n: int, modulus_chain, scale_bits: int, level: int,
                 layout: str = "reference"):
        self.n = n
        self.layout = layout
        two_n = 2 * n
        chain = tuple(modulus_chain)
        used: set = set()
        nominal = float(2**scale_bits)
        rescale = [None] * level
        scale_at = [0.0] * (level + 1)
        scale_at[level] = nominal
        if layout == "reference":
            base = primes_for_product(2.0 ** chain[0], two_n, used)
            special = primes_for_product(2.0 ** chain[-1], two_n, used)
            for lv in range(level, 0, -1):
                entry = primes_for_product(scale_at[lv] ** 2 / nominal, two_n, used)
                rescale[lv - 1] = entry
                scale_at[lv - 1] = scale_at[lv] ** 2 / math.prod(entry)
        elif layout in ("baseline", "schedule"):
            def wide(bits):
                k = max(1, -(-bits // 60))
                out = []
                for _ in range(k):
                    p = largest_ntt_prime_below(bits // k, two_n, used)
                    used.add(p)
                    out.append(p)
                return out
            base = wide(chain[0])
            special = wide(chain[-1])
            for lv in range(level, 0, -1):
                if layout == "baseline":
                    p = largest_ntt_prime_below(chain[lv], two_n, used)
                else:
                    target = scale_at[lv] ** 2 / nominal
                    p = nearest_ntt_prime(round(target), two_n, used, max_bits=61)
                used.add(p)
                rescale[lv - 1] = [p]
                scale_at[lv - 1] = scale_at[lv] ** 2 / p
        else:
            raise OracleError(f"unknown layout {layout}")
        self.entry_primes = [base] + rescale + [special]
        self.primes = base + [p for e in rescale for p in e]
        self.special_primes = special
        self.all_primes = self.primes + special
        self.plans = {p: NttPlan(p, n) for p in self.all_primes}
        self.level_limbs = [len(base)]
        for e in rescale:
            self.level_limbs.append(self.level_limbs[-1] + len(e))
        self.entry_products = [math.prod(e) for e in self.entry_primes]
        self.special_product = math.prod(special)
        self.scale_at = scale_at

    def limbs_at(self, level: int) -> list:
        return self.primes[: self.level_limbs[level]]

    def modulus_at(self, level: int) -> int:
        return math.prod(self.limbs_at(level))


# ---------------------------------------------------------------------------
# ring elements (ring.py:62-136): planes = list of 1-D arrays, one per prime
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class Elem:
    primes: tuple
    planes: list
    ntt: bool = False

    def copy(self):
        return Elem(self.primes, [p.copy() for p in self.planes], self.ntt)

    def to_u64(self) -> np.ndarray:
        return np.stack([np.asarray(pl, dtype=object).astype(np.uint64) if pl.dtype == object
                         else pl.astype(np.uint64) for pl in self.planes])


def _P(p):
    return np.uint64(p) if p < (1 << 31) else p


def _obj(plane) -> np.ndarray:
    """A limb as an object array of exact Python ints (vectorised big-int math)."""
    return np.array([int(v) for v in plane.tolist()], dtype=object)


def _centered(plane, q: int) -> np.ndarray:
    """Centred representative of residues mod q (keys.py:85-89, ring.py:171-175:
    values above q // 2 map to v - q), as Python ints."""
    d = _obj(plane)
    return np.where(d > q // 2, d - q, d)


def e_add(a: Elem, b: Elem) -> Elem:
    assert a.primes == b.primes and a.ntt == b.ntt
    return Elem(a.primes, [(x + y) % _P(p) for x, y, p in zip(a.planes, b.planes, a.primes)], a.ntt)


def e_sub(a: Elem, b: Elem) -> Elem:
    assert a.primes == b.primes and a.ntt == b.ntt
    return Elem(a.primes, [(x + (_P(p) - y)) % _P(p) for x, y, p in zip(a.planes, b.planes, a.primes)],
                a.ntt)


def e_neg(a: Elem) -> Elem:
    return Elem(a.primes, [(_P(p) - x) % _P(p) for x, p in zip(a.planes, a.primes)], a.ntt)


def e_scalar(a: Elem, value: int) -> Elem:
    return Elem(a.primes, [x * _P(value % p) % _P(p) for x, p in zip(a.planes, a.primes)], a.ntt)


def e_mul(a: Elem, b: Elem, chain: Chain) -> Elem:
    a, b = e_ntt(a, chain), e_ntt(b, chain)
    assert a.primes == b.primes
    return Elem(a.primes, [x * y % _P(p) for x, y, p in zip(a.planes, b.planes, a.primes)], True)


def e_ntt(a: Elem, chain: Chain) -> Elem:
    if a.ntt:
        return a
    return Elem(a.primes, [chain.plans[p].forward(x) for x, p in zip(a.planes, a.primes)], True)


def e_coeff(a: Elem, chain: Chain) -> Elem:
    if not a.ntt:
        return a
    return Elem(a.primes, [chain.plans[p].inverse(x) for x, p in zip(a.planes, a.primes)], False)


def e_restrict(a: Elem, primes) -> Elem:
    primes = tuple(primes)
    return Elem(primes, [a.planes[a.primes.index(p)].copy() for p in primes], a.ntt)


def make_element(primes, coeffs: np.ndarray) -> Elem:
    """ring.py:139-145 (signed integers -> residues)."""
    vals = [int(v) for v in np.asarray(coeffs).tolist()]
    planes = [as_limb([v % p for v in vals], p) for p in primes]
    return Elem(tuple(primes), planes, False)


def divide_round_by_prime(a: Elem, drop: int) -> Elem:
    """ring.py:165-183: exact centered divide-and-round by one limb."""
    assert not a.ntt
    di = a.primes.index(drop)
    digit = _centered(a.planes[di], drop)
    keep = [i for i in range(len(a.primes)) if i != di]
    primes = tuple(a.primes[i] for i in keep)
    out = []
    for i in keep:
        p = a.primes[i]
        r = as_limb(digit % p, p)
        inv = pow(drop, -1, p)
        out.append((a.planes[i] + (_P(p) - r)) % _P(p) * _P(inv) % _P(p))
    return Elem(primes, out, False)


def divide_round_by_primes(a: Elem, drops) -> Elem:
    for p in drops:
        a = divide_round_by_prime(a, p)
    return a


def lift_centered(a: Elem, chain: Chain) -> list:
    """ring.py:192-208 via Python ints (CRT then center)."""
    a = e_coeff(a, chain)
    Q = math.prod(a.primes)
    out = []
    cols = [[int(v) for v in pl.tolist()] for pl in a.planes]
    # Garner
    n = len(cols[0])
    x = cols[0][:]
    mod = a.primes[0]
    for i in range(1, len(a.primes)):
        p = a.primes[i]
        inv = pow(mod % p, -1, p)
        for k in range(n):
            t = (cols[i][k] - x[k] % p) % p * inv % p
            x[k] += t * mod
        mod *= p
    half = Q // 2
    for v in x:
        out.append(v - Q if v > half else v)
    return out


def automorphism_tables(n: int, galois: int):
    """ring.py:211-219."""
    idx = np.arange(n, dtype=np.int64)
    exp = (idx * galois) % (2 * n)
    return exp % n, np.where(exp >= n, -1, 1)


def apply_automorphism(a: Elem, galois: int) -> Elem:
    """ring.py:222-232."""
    assert not a.ntt
    n = len(a.planes[0])
    target, sign = automorphism_tables(n, galois)
    out = []
    for x, p in zip(a.planes, a.primes):
        P = _P(p)
        flipped = x.copy()
        neg = sign < 0
        flipped[neg] = (P - x[neg]) % P
        plane = x.copy()
        plane[target] = flipped
        out.append(plane)
    return Elem(a.primes, out, False)


# ---------------------------------------------------------------------------
# encoder (encoding.py:17-76)
# ---------------------------------------------------------------------------


class Encoder:
    def __init__(self, n: int):
        self.n = n
        slots = n // 2
        exps = np.empty(slots, dtype=np.int64)
        e = 1
        for i in range(slots):
            exps[i] = e
            e = (e * 5) % (2 * n)
        self.bins = (exps - 1) // 2
        self.conj_bins = (2 * n - exps - 1) // 2
        j = np.arange(n)
        self.psi_pow = np.exp(1j * np.pi * j / n)
        self.psi_inv_pow = np.conj(self.psi_pow)

    def embed(self, values, scale: float) -> np.ndarray:
        slots = self.n // 2
        v = np.zeros(slots)
        vals = np.asarray(values, dtype=np.float64)
        v[: vals.shape[0]] = vals
        spec = np.zeros(self.n, dtype=np.complex128)
        scaled = v * scale
        spec[self.bins] = scaled
        spec[self.conj_bins] = scaled
        w = np.fft.fft(spec) / self.n
        coeffs = np.rint(np.real(w * self.psi_inv_pow))
        if np.max(np.abs(coeffs)) >= MAX_SAFE_COEFF:
            raise EncodingOverflowError("coefficients exceed 2^52")
        return coeffs.astype(np.int64)

    def unembed(self, coeffs, scale: float) -> np.ndarray:
        w = np.asarray(coeffs, dtype=np.float64) * self.psi_pow
        spec = np.fft.ifft(w) * self.n
        return np.real(spec[self.bins]) / scale


# ---------------------------------------------------------------------------
# keys (keys.py:29-142), generalised to digits of alpha limbs
# ---------------------------------------------------------------------------


def sample_uniform(primes, rng, n) -> list:
    """ring.py:148-153."""
    out = []
    for p in primes:
        if p < (1 << 63):
            out.append(as_limb(rng.integers(0, p, n, dtype=np.uint64), p))
    return out


def sample_gaussian(rng, n, sigma=ERROR_SIGMA) -> np.ndarray:
    """ring.py:156-158."""
    return np.rint(rng.normal(0.0, sigma, n)).astype(np.int64)


def sample_ternary(rng, n) -> np.ndarray:
    """ring.py:161-162."""
    return rng.integers(-1, 2, n).astype(np.int64)


@dataclasses.dataclass
class KSKey:
    rows_b: list  # list of Elem over all primes, NTT domain
    rows_a: list


def digit_ranges(n_limbs: int, alpha: int):
    return [(j, min(j + alpha, n_limbs)) for j in range(0, n_limbs, alpha)]


def make_keyswitch_key(chain: Chain, s_full: Elem, source_ntt: Elem, rng, alpha: int = 1) -> KSKey:
    """keys.py:49-71; row j carries P*source on the limbs of digit j."""
    full = chain.all_primes
    n = chain.n
    P = chain.special_product
    rows_b, rows_a = [], []
    for lo, hi in digit_ranges(len(chain.primes), alpha):
        a = Elem(tuple(full), sample_uniform(full, rng, n), True)
        e = e_ntt(make_element(full, sample_gaussian(rng, n)), chain)
        b = e_add(e_neg(e_mul(a, s_full, chain)), e)
        for i in range(lo, hi):
            q = chain.primes[i]
            k = full.index(q)
            msg = source_ntt.planes[k] * _P(P % q) % _P(q)
            b.planes[k] = (b.planes[k] + msg) % _P(q)
        rows_b.append(b)
        rows_a.append(a)
    return KSKey(rows_b, rows_a)


def modup_digit(d: Elem, lo: int, hi: int, ext, centered: bool = True) -> Elem:
    """Digit [lo, hi) of d (coefficient domain) lifted into the ext basis.

    centered (alpha == 1): the reference's centered digit (keys.py:85-89).
    otherwise (alpha > 1, including a short last digit): fast basis conversion
               y_i = [x_i * qhat_i^-1]_{q_i}, out_p = sum_i y_i * [qhat_i]_p
               (the digit's own limbs are copied).
    """
    if centered:
        assert hi - lo == 1
        q = d.primes[lo]
        digit = _centered(d.planes[lo], q)
        planes = []
        for p in ext:
            if p == q:
                planes.append(d.planes[lo].copy())
            else:
                planes.append(as_limb(digit % p, p))
        return Elem(tuple(ext), planes, False)
    qs = d.primes[lo:hi]
    Qj = math.prod(qs)
    ys = []
    for i, q in enumerate(qs):
        qhat = Qj // q
        inv = pow(qhat % q, -1, q)
        ys.append(_obj(d.planes[lo + i]) * inv % q)
    planes = []
    for p in ext:
        if p in qs:
            planes.append(d.planes[d.primes.index(p)].copy())
            continue
        acc = sum(y * ((Qj // q) % p) for y, q in zip(ys, qs))
        planes.append(as_limb(acc % p, p))
    return Elem(tuple(ext), planes, False)


def key_switch(chain: Chain, d: Elem, key: KSKey, alpha: int = 1):
    """keys.py:74-100 generalised to digits of alpha limbs."""
    d = e_coeff(d, chain)
    current = list(d.primes)
    ext = tuple(current + chain.special_primes)
    acc_b = acc_a = None
    for j, (lo, hi) in enumerate(digit_ranges(len(current), alpha)):
        dig = e_ntt(modup_digit(d, lo, hi, ext, centered=(alpha == 1)), chain)
        kb = e_restrict(key.rows_b[j], ext)
        ka = e_restrict(key.rows_a[j], ext)
        tb, ta = e_mul(dig, kb, chain), e_mul(dig, ka, chain)
        acc_b = tb if acc_b is None else e_add(acc_b, tb)
        acc_a = ta if acc_a is None else e_add(acc_a, ta)
    drops = list(reversed(chain.special_primes))
    out_b = divide_round_by_primes(e_coeff(acc_b, chain), drops)
    out_a = divide_round_by_primes(e_coeff(acc_a, chain), drops)
    return out_b, out_a


# ---------------------------------------------------------------------------
# ciphertext-level operations (backend.py:50-206)
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class Ct:
    c0: Elem
    c1: Elem
    level: int


class OracleCkks:
    """Restatement of CkksBackend's payload semantics (backend.py:50-206).

    ``serial`` bookkeeping is left to the caller: encrypt takes the serial the
    reference would pass to default_rng((seed, serial)) (backend.py:174).
    """

    def __init__(self, n, modulus_chain, scale_bits, level, rotation_steps=(), rng_seed=0,
                 layout="reference", alpha=1, secret=None, refresh_level=None):
        self.chain = Chain(n, modulus_chain, scale_bits, level, layout)
        self.n = n
        self.level = level
        self.alpha = alpha
        self.refresh_level = level if refresh_level is None else refresh_level
        self.encoder = Encoder(n)
        self.rng_seed = rng_seed
        rng = np.random.default_rng(rng_seed)
        full = self.chain.all_primes
        coeffs = sample_ternary(rng, n)  # keys.py:40 (always consumed)
        if secret is not None:
            coeffs = np.asarray(secret, dtype=np.int64)
        self.secret = coeffs
        self.s_full = e_ntt(make_element(full, coeffs), self.chain)
        self.relin = make_keyswitch_key(self.chain, self.s_full,
                                        e_mul(self.s_full, self.s_full, self.chain), rng, alpha)
        self.rot_keys = {}
        self.galois_for_step = {}
        slots = n // 2
        for step in sorted({k % slots for k in rotation_steps} - {0}):
            g = pow(5, step, 2 * n)
            self.galois_for_step[step] = g
            s_rot = e_ntt(apply_automorphism(e_coeff(self.s_full, self.chain), g), self.chain)
            self.rot_keys[g] = make_keyswitch_key(self.chain, self.s_full, s_rot, rng, alpha)
        self.bs_rng = np.random.default_rng(rng_seed + 0x5EED)

    # -- helpers
    def scale(self, level):
        return self.chain.scale_at[level]

    def s_restricted(self, primes):
        return e_restrict(self.s_full, primes)

    def rescale(self, ct: Ct) -> Ct:
        """backend.py:86-92."""
        drops = list(reversed(self.chain.entry_primes[ct.level]))
        return Ct(divide_round_by_primes(e_coeff(ct.c0, self.chain), drops),
                  divide_round_by_primes(e_coeff(ct.c1, self.chain), drops), ct.level - 1)

    def adjust(self, ct: Ct, target: int) -> Ct:
        """backend.py:94-112."""
        if ct.level == target:
            return ct
        origin = self.scale(ct.level)
        staging = target + 1
        primes = tuple(self.chain.limbs_at(staging))
        c0, c1 = e_restrict(ct.c0, primes), e_restrict(ct.c1, primes)
        factor = self.adjust_factor(ct.level, target)
        return self.rescale(Ct(e_scalar(c0, factor), e_scalar(c1, factor), staging))

    def adjust_factor(self, origin_level, target) -> int:
        s_star = self.scale(target) * self.chain.entry_products[target + 1] / self.scale(origin_level)
        return int(np.rint(s_star))

    def encode(self, values, level) -> Elem:
        coeffs = self.encoder.embed(values, self.scale(level))
        bound = float(np.max(np.abs(coeffs)))
        if 4.0 * bound >= float(self.chain.modulus_at(level)):
            raise EncodingOverflowError("no headroom")
        return make_element(self.chain.limbs_at(level), coeffs)

    def encrypt_coeffs(self, m: Elem, level: int, serial: int) -> Ct:
        """backend.py:173-182 with the plaintext already encoded."""
        rng = np.random.default_rng((self.rng_seed, serial))
        primes = self.chain.limbs_at(level)
        a = Elem(tuple(primes), sample_uniform(primes, rng, self.n), True)
        e = make_element(primes, sample_gaussian(rng, self.n))
        s = self.s_restricted(tuple(primes))
        c0 = e_add(e_add(e_coeff(e_neg(e_mul(a, s, self.chain)), self.chain), m), e)
        return Ct(c0, e_coeff(a, self.chain), level)

    def encrypt(self, values, level, serial) -> Ct:
        return self.encrypt_coeffs(self.encode(values, level), level, serial)

    def phase(self, ct: Ct) -> Elem:
        s = self.s_restricted(ct.c0.primes)
        return e_add(e_coeff(ct.c0, self.chain), e_coeff(e_mul(ct.c1, s, self.chain), self.chain))

    def decrypt(self, ct: Ct) -> np.ndarray:
        """backend.py:187-190."""
        coeffs = lift_centered(self.phase(ct), self.chain)
        return self.encoder.unembed(np.array([float(c) for c in coeffs]), self.scale(ct.level))

    def add(self, a: Ct, b: Ct, sub=False) -> Ct:
        lvl = min(a.level, b.level)
        a, b = self.adjust(a, lvl), self.adjust(b, lvl)
        f = e_sub if sub else e_add
        return Ct(f(e_coeff(a.c0, self.chain), e_coeff(b.c0, self.chain)),
                  f(e_coeff(a.c1, self.chain), e_coeff(b.c1, self.chain)), lvl)

    def mul(self, a: Ct, b: Ct) -> Ct:
        """backend.py:136-143."""
        lvl = min(a.level, b.level)
        a, b = self.adjust(a, lvl), self.adjust(b, lvl)
        ch = self.chain
        a0, a1, b0, b1 = (e_ntt(x, ch) for x in (a.c0, a.c1, b.c0, b.c1))
        d0 = e_mul(a0, b0, ch)
        d1 = e_add(e_mul(a0, b1, ch), e_mul(a1, b0, ch))
        d2 = e_mul(a1, b1, ch)
        r0, r1 = key_switch(ch, d2, self.relin, self.alpha)
        full = Ct(e_add(e_coeff(d0, ch), r0), e_add(e_coeff(d1, ch), r1), lvl)
        return self.rescale(full)

    def mul_plain_coeffs(self, a: Ct, m: Elem) -> Ct:
        """backend.py:147-151 with the plaintext already encoded at a.level."""
        ch = self.chain
        pt = e_ntt(m, ch)
        return self.rescale(Ct(e_coeff(e_mul(a.c0, pt, ch), ch), e_coeff(e_mul(a.c1, pt, ch), ch),
                               a.level))

    def add_plain_coeffs(self, a: Ct, m: Elem) -> Ct:
        """backend.py:152-153 (sub passes the encoding of -values)."""
        return Ct(e_add(e_coeff(a.c0, self.chain), m), a.c1.copy(), a.level)

    def rotate(self, a: Ct, k: int) -> Ct:
        """backend.py:155-171 (k already normalised to [1, N/2))."""
        g = pow(5, k, 2 * self.n)
        key = self.rot_keys[g]
        ch = self.chain
        c0r = apply_automorphism(e_coeff(a.c0, ch), g)
        c1r = apply_automorphism(e_coeff(a.c1, ch), g)
        r0, r1 = key_switch(ch, c1r, key, self.alpha)
        return Ct(e_add(c0r, r0), r1, a.level)


def ct_to_u64(ct: Ct, chain: Chain) -> np.ndarray:
    """[2][limbs][N] uint64 in the coefficient domain (RBCT plane order)."""
    return np.stack([e_coeff(ct.c0, chain).to_u64(), e_coeff(ct.c1, chain).to_u64()])


def ct_from_u64(arr: np.ndarray, level: int, chain: Chain) -> Ct:
    primes = tuple(chain.limbs_at(level))
    c = [Elem(primes, [as_limb(arr[i, j], p) for j, p in enumerate(primes)], False) for i in range(2)]
    return Ct(c[0], c[1], level)
