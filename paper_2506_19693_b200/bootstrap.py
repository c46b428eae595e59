"""Full-slot CKKS bootstrapping on the B200 backend (BASELINE config 3).

The reference's "bootstrap" is a custodian refresh (decrypt + re-encrypt,
ckks/backend.py:195-206); this is the homomorphic procedure the paper's
implementation uses, built from the backend's kernels:

  1. ModRaise       level-0 ciphertext reinterpreted modulo Q_L (centred lift)
  2. CoeffToSlot    P V^-1 as `levels` BSGS linear transforms (hoisted baby-step
                    rotations, one rescale per giant step), scaled so the slots
                    hold (c + q0 I) / (q0 (K+1)) (bit-reversed order)
  3. real/imag      conjugation key: Re = ct + conj(ct) (the 1/2 is folded into
                    CoeffToSlot), Im = (ct - conj(ct)) * (-X^{N/2})
  4. EvalMod        Chebyshev interpolant (degree 119) of cos(2π((K+1)x - 1/4)/2^r)
                    evaluated with baby steps T_0..T_15 and giant steps
                    T_16, T_32, T_64, then r = 2 double-angle steps -> sin(2π u)
  5. recombine      Re + X^{N/2} Im
  6. SlotToCoeff    V P, with the 1/(2π) and q0/Δ factors folded in
and finally aligns to params.refresh_level.  Constants: bootstrap_consts.py.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import bootstrap_consts as BC
from .backend import GpuCiphertext


def bootstrap_rotations(params, levels: int = 3) -> set:
    """Rotation steps the CoeffToSlot / SlotToCoeff BSGS plans need."""
    slots = params.slot_count
    two_n = 2 * params.poly_degree
    rots = set()
    for inverse in (True, False):
        for m in BC.grouped_transform(slots, two_n, levels, inverse):
            rots |= BC.bsgs_rotations(BC.bsgs_plan(m, slots), slots)
    return rots


class Bootstrapper:
    def __init__(self, backend, K: int = 28, r: int = 2, degree: int = 119, levels: int = 3):
        be = self.be = backend
        ch = be.chain
        self.K, self.r, self.degree, self.levels = K, r, degree, levels
        n = be.n
        slots = n // 2
        self.slots = slots
        L = be.params.level
        q0 = ch.entry_products[0]
        self.q0 = q0
        cts = BC.grouped_transform(slots, 2 * n, levels, inverse=True)
        stc = BC.grouped_transform(slots, 2 * n, levels, inverse=False)
        # CtS overall scalar: value_L = V (c + q0 I)'/scale_L  ->  (c + q0 I)'/(2 q0 (K+1))
        kappa = ch.scale_at[L] / (2.0 * q0 * (K + 1)) / slots
        k_lvl = abs(kappa) ** (1.0 / levels)
        cts = [{k: v * k_lvl for k, v in m.items()} for m in cts]
        self.cts_plans = [BC.bsgs_plan(m, slots) for m in cts]
        # StC overall scalar sigma = q0 / (2π scale_0), spread over the levels
        sigma = q0 / (2.0 * math.pi * ch.scale_at[0])
        s_lvl = sigma ** (1.0 / levels)
        self.stc_plans = [BC.bsgs_plan({k: v * s_lvl for k, v in m.items()}, slots) for m in stc]
        self.cheb = BC.cheb_coeffs(BC.evalmod_function(K, r), degree)
        self._pt_cache: dict = {}
        self._const_cache: dict = {}
        two_n = 2 * n
        self.conj = two_n - 1

    # -- plaintext caches ------------------------------------------------------
    def _pt(self, tag, level, z):
        key = (tag, level)
        hit = self._pt_cache.get(key)
        if hit is None:
            hit = self._pt_cache[key] = self.be.encode_complex_ntt(z, level)
        return hit

    def _galois(self, step: int) -> int:
        return pow(5, step % self.slots, 2 * self.be.n)

    # -- homomorphic building blocks on (data, level) pairs ----------------------
    def _align(self, a, b):
        (da, la), (db, lb) = a, b
        if la > lb:
            da, la = self.be._adjust_data(da, la, lb), lb
        elif lb > la:
            db, lb = self.be._adjust_data(db, lb, la), la
        return da, db, la

    def _add(self, a, b):
        da, db, lvl = self._align(a, b)
        return self.be.chain.add(da, db, self.be._limbs(lvl)), lvl

    def _sub(self, a, b):
        da, db, lvl = self._align(a, b)
        return self.be.chain.sub(da, db, self.be._limbs(lvl)), lvl

    def _mul(self, a, b):
        da, db, lvl = self._align(a, b)
        out = self.be._hmult(da.unsqueeze(0).contiguous(), db.unsqueeze(0).contiguous(), lvl)
        return out[0], lvl - 1

    def _mul_const(self, a, c: float):
        da, lvl = a
        key = (float(c), lvl)
        pt = self._const_cache.get(key)
        if pt is None:
            pt = self._const_cache[key] = self.be._encode_rns(np.full(self.slots, c), lvl, ntt=True)
        m = self.be._limbs(lvl)
        return self.be._rescale_data(self.be.chain.mul(da, pt, m, b_rows=m), lvl), lvl - 1

    def _add_const(self, a, c: float):
        da, lvl = a
        m = self.be._limbs(lvl)
        pt = self.be._encode_rns(np.full(self.slots, c), lvl, ntt=True)
        out = da.clone()
        self.be.chain.add(da[0], pt, m, out=out[0])
        return out, lvl

    def _double(self, a):
        da, lvl = a
        return self.be.chain.add(da, da, self.be._limbs(lvl)), lvl

    # -- linear transforms ------------------------------------------------------------
    def _linear(self, x, plan, tag):
        """sum_g rot(sum_b pt_gb * rot(x, b s), g n1 s) with hoisted baby steps."""
        be, ch = self.be, self.be.chain
        data, lvl = x
        s, n1, rows = plan
        m = be._limbs(lvl)
        babies = sorted({b for row in rows.values() for b in row if b})
        rots = dict(zip(babies, be.hoisted_rotations(data, lvl, [self._galois(b * s)
                                                                 for b in babies])))
        rots[0] = data
        acc = None
        for g, row in sorted(rows.items()):
            inner = None
            for b, diag in row.items():
                pt = self._pt((tag, g, b), lvl, diag)
                term = ch.mul(rots[b], pt, m, b_rows=m)
                inner = term if inner is None else ch.add(inner, term, m, out=inner)
            inner = be._rescale_data(inner, lvl)
            if g:
                inner = be.rotate_data(inner, lvl - 1, self._galois(g * n1 * s))
            acc = inner if acc is None else ch.add(acc, inner, be._limbs(lvl - 1), out=acc)
        return acc, lvl - 1

    # -- EvalMod ------------------------------------------------------------------
    def _chebyshev_basis(self, x):
        T = {1: x}

        def get(k):
            if k in T:
                return T[k]
            if k % 2 == 0:
                h = get(k // 2)
                T[k] = self._add_const(self._double(self._mul(h, h)), -1.0)
            else:
                a, b = get(k // 2), get(k // 2 + 1)
                T[k] = self._sub(self._double(self._mul(a, b)), get(1))
            return T[k]

        for k in range(2, 17):
            get(k)
        get(32)
        get(64)
        return T

    def _eval_cheb(self, c, T):
        c = np.asarray(c, dtype=np.float64)
        deg = len(c) - 1
        while deg > 0 and abs(c[deg]) < 1e-300:
            deg -= 1
        c = c[: deg + 1]
        if deg < 16:
            acc = None
            for k in range(1, deg + 1):
                if abs(c[k]) < 1e-18:
                    continue
                term = self._mul_const(T[k], c[k])
                acc = term if acc is None else self._add(acc, term)
            if acc is None:
                acc = self._mul_const(T[1], 0.0)
            return self._add_const(acc, c[0])
        n = 1 << (deg.bit_length() - 1)
        q = np.zeros(deg - n + 1)
        q[0] = c[n]
        q[1:] = 2.0 * c[n + 1:]
        rem = c[:n].copy()
        for j in range(1, deg - n + 1):
            rem[n - j] -= c[n + j]
        return self._add(self._mul(self._eval_cheb(q, T), T[n]), self._eval_cheb(rem, T))

    def _evalmod(self, x):
        T = self._chebyshev_basis(x)
        y = self._eval_cheb(self.cheb, T)
        for _ in range(self.r):
            y = self._add_const(self._double(self._mul(y, y)), -1.0)
        return y

    # -- the whole procedure ----------------------------------------------------------
    def bootstrap(self, ct: GpuCiphertext) -> GpuCiphertext:
        be, ch = self.be, self.be.chain
        raised = be.mod_raise(ct)
        x = (raised.data, raised.level)
        for t, plan in enumerate(self.cts_plans):
            x = self._linear(x, plan, ("cts", t))
        data, lvl = x
        m = be._limbs(lvl)
        conj = be.rotate_data(data, lvl, self.conj)
        re = (ch.add(data, conj, m), lvl)
        diff = ch.sub(data, conj, m)
        mono = be.monomial_ntt(3 * be.n // 2, lvl)  # -X^{N/2} = X^{3N/2}
        im = (ch.mul(diff, mono, m, b_rows=m), lvl)
        y_re = self._evalmod(re)
        y_im = self._evalmod(im)
        d_im, l_im = y_im
        y_im = (ch.mul(d_im, be.monomial_ntt(be.n // 2, l_im), be._limbs(l_im),
                       b_rows=be._limbs(l_im)), l_im)
        z = self._add(y_re, y_im)
        for t, plan in enumerate(self.stc_plans):
            z = self._linear(z, plan, ("stc", t))
        data, lvl = z
        rl = be.params.refresh_level
        if lvl > rl:
            data, lvl = be._adjust_data(data, lvl, rl), rl
        if lvl < rl:
            raise RuntimeError(f"bootstrapping consumed too many levels ({lvl} < {rl})")
        return GpuCiphertext(data, lvl)
