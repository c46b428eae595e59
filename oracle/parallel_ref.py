"""Multi-core CPU timing of the reference HMult — TEST/BENCH INFRASTRUCTURE ONLY.

bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm time the
reference's own algorithm (ckks/backend.py:136-143 -> keys.py:74-100, as
restated in oracle/ckks_oracle.py) with every host core: the key-switch
inner loop is split by extended limb (each process owns a disjoint slice of
the Q u P limbs, runs every digit's lift + NTT + key multiply-accumulate for
those limbs and writes its slice of the accumulator into shared memory); the
tensor product, the final iNTT and the divide-and-round run in the parent.
Inputs and the per-limb NTT plans are inherited through fork, so nothing is
pickled but the limb index lists.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import ckks_oracle as O

_STATE: dict = {}


def _worker(limb_ids):
    st = _STATE
    chain, d2, key_b, key_a, ext = st["chain"], st["d2"], st["kb"], st["ka"], st["ext"]
    out = np.ndarray(st["shape"], dtype=np.uint64, buffer=st["shm"].buf)
    primes_q = d2.primes
    for e in limb_ids:
        p = ext[e]
        P = np.uint64(p)
        plan = chain.plans[p]
        acc_b = np.zeros(chain.n, dtype=np.uint64)
        acc_a = np.zeros(chain.n, dtype=np.uint64)
        for i, q in enumerate(primes_q):
            x = d2.planes[i].astype(np.int64)
            if p == q:
                dig = d2.planes[i]
            else:
                x[x > q // 2] -= q
                dig = (x % p).astype(np.uint64)
            f = plan.forward(dig)
            acc_b = (acc_b + f * key_b[i][e] % P) % P
            acc_a = (acc_a + f * key_a[i][e] % P) % P
        out[0, e] = acc_b
        out[1, e] = acc_a
    return len(limb_ids)


def make_random_case(n: int, entries: int, seed: int):
    """Chain of `entries` 40-bit entries (+ one 60-bit special) in the
    reference prime layout, two random ciphertexts at the top level and random
    key rows (their values do not change the work)."""
    chain = O.Chain(n, (40,) * entries + (60,), 40, entries - 1, "reference")
    rng = np.random.default_rng(seed)
    lvl = entries - 1
    prim = chain.limbs_at(lvl)
    full = chain.all_primes

    def rand(primes, ntt):
        return O.Elem(tuple(primes), [rng.integers(0, p, n, dtype=np.uint64) for p in primes], ntt)

    cts = [O.Ct(rand(prim, False), rand(prim, False), lvl) for _ in range(2)]
    kb = rand(full, True)
    ka = rand(full, True)
    return chain, cts, kb, ka


def hmult_parallel(chain, a: "O.Ct", b: "O.Ct", kb_row: "O.Elem", ka_row: "O.Elem",
                   procs: int) -> tuple:
    """One HMult, reference algorithm, `procs` processes.  The same random key
    row stands in for every digit's row.  Returns (Ct, seconds)."""
    from multiprocessing import shared_memory

    t0 = time.perf_counter()
    ch = chain
    a0, a1, b0, b1 = (O.e_ntt(x, ch) for x in (a.c0, a.c1, b.c0, b.c1))
    d0 = O.e_mul(a0, b0, ch)
    d1 = O.e_add(O.e_mul(a0, b1, ch), O.e_mul(a1, b0, ch))
    d2 = O.e_coeff(O.e_mul(a1, b1, ch), ch)
    ext = list(d2.primes) + list(ch.special_primes)
    full = ch.all_primes
    kb = [[kb_row.planes[full.index(p)] for p in ext]] * len(d2.primes)
    ka = [[ka_row.planes[full.index(p)] for p in ext]] * len(d2.primes)
    shape = (2, len(ext), ch.n)
    shm = shared_memory.SharedMemory(create=True, size=int(np.prod(shape)) * 8)
    try:
        _STATE.update(chain=ch, d2=d2, kb=kb, ka=ka, ext=ext, shape=shape, shm=shm)
        parts = [list(range(len(ext)))[i::procs] for i in range(procs)]
        parts = [p for p in parts if p]
        if procs > 1:
            with mp.get_context("fork").Pool(len(parts)) as pool:
                pool.map(_worker, parts)
        else:
            _worker(parts[0])
        acc = np.ndarray(shape, dtype=np.uint64, buffer=shm.buf).copy()
    finally:
        _STATE.clear()
        shm.close()
        shm.unlink()
    acc_b = O.Elem(tuple(ext), [acc[0, e] for e in range(len(ext))], True)
    acc_a = O.Elem(tuple(ext), [acc[1, e] for e in range(len(ext))], True)
    drops = list(reversed(ch.special_primes))
    r0 = O.divide_round_by_primes(O.e_coeff(acc_b, ch), drops)
    r1 = O.divide_round_by_primes(O.e_coeff(acc_a, ch), drops)
    full_ct = O.Ct(O.e_add(O.e_coeff(d0, ch), r0), O.e_add(O.e_coeff(d1, ch), r1), a.level)
    drops = list(reversed(ch.entry_primes[a.level]))
    out = O.Ct(O.divide_round_by_primes(full_ct.c0, drops),
               O.divide_round_by_primes(full_ct.c1, drops), a.level - 1)
    return out, time.perf_counter() - t0


def _key_switch_parallel(ch, d2, kb_row, ka_row, procs):
    """keys.py:74-100 for the coefficient-domain polynomial d2: the per-limb
    digit lift + NTT + key multiply-accumulate split over `procs` processes,
    then iNTT and the sequential divide-round by the special primes."""
    from multiprocessing import shared_memory

    ext = list(d2.primes) + list(ch.special_primes)
    full = ch.all_primes
    kb = [[kb_row.planes[full.index(p)] for p in ext]] * len(d2.primes)
    ka = [[ka_row.planes[full.index(p)] for p in ext]] * len(d2.primes)
    shape = (2, len(ext), ch.n)
    shm = shared_memory.SharedMemory(create=True, size=int(np.prod(shape)) * 8)
    try:
        _STATE.update(chain=ch, d2=d2, kb=kb, ka=ka, ext=ext, shape=shape, shm=shm)
        parts = [list(range(len(ext)))[i::procs] for i in range(procs)]
        parts = [p for p in parts if p]
        if procs > 1:
            with mp.get_context("fork").Pool(len(parts)) as pool:
                pool.map(_worker, parts)
        else:
            _worker(parts[0])
        acc = np.ndarray(shape, dtype=np.uint64, buffer=shm.buf).copy()
    finally:
        _STATE.clear()
        shm.close()
        shm.unlink()
    acc_b = O.Elem(tuple(ext), [acc[0, e] for e in range(len(ext))], True)
    acc_a = O.Elem(tuple(ext), [acc[1, e] for e in range(len(ext))], True)
    drops = list(reversed(ch.special_primes))
    return (O.divide_round_by_primes(O.e_coeff(acc_b, ch), drops),
            O.divide_round_by_primes(O.e_coeff(acc_a, ch), drops))


def hrot_parallel(chain, a: "O.Ct", galois: int, kb_row: "O.Elem", ka_row: "O.Elem",
                  procs: int) -> tuple:
    """One rotation, reference algorithm (backend.py:155-171): automorphism of
    both components, key switch of c1', (c0' + r0, r1).  Returns (Ct, seconds)."""
    t0 = time.perf_counter()
    c0 = O.apply_automorphism(a.c0, galois)
    c1 = O.apply_automorphism(a.c1, galois)
    r0, r1 = _key_switch_parallel(chain, c1, kb_row, ka_row, procs)
    out = O.Ct(O.e_add(c0, r0), r1, a.level)
    return out, time.perf_counter() - t0


def default_procs() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1
