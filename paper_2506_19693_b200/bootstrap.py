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

import contextlib
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
    """Values inside are (data [B, 2, m, N] NTT domain, level, scale) triples
    (B ciphertexts bootstrapped together; one ciphertext is B = 1): the
    bootstrapping levels (prime_layout="bootstrap": ~60-bit primes above the
    refresh level) run at scale ~q0 ≈ 2^60 with every plaintext encoded at the
    prime it is about to be divided by, so the noise floor is ~2^-45 of the
    O(1) slot values while the user scale stays 2^scale_bits below."""

    def __init__(self, backend, K: int = 28, r: int = 2, degree: int = 119, levels: int = 3):
        be = self.be = backend
        ch = be.chain
        self.K, self.r, self.degree, self.levels = K, r, degree, levels
        # side streams for the giant rows of small batches (see _linear)
        self.streams, self.stream_batch_max = 3, 4
        self._side = [torch.cuda.Stream(be.device) for _ in range(self.streams)]
        n = be.n
        slots = n // 2
        self.slots = slots
        self.q0 = ch.entry_products[0]
        cts = BC.grouped_transform(slots, 2 * n, levels, inverse=True)
        stc = BC.grouped_transform(slots, 2 * n, levels, inverse=False)
        # raised ct read at scale q0 has slots V u', u = (c + q0 I)/q0; CoeffToSlot
        # maps them to P u' / (2 (K+1)) (the 1/2 pairs with ct + conj(ct))
        k_lvl = (1.0 / (2.0 * (K + 1) * slots)) ** (1.0 / levels)
        self.cts_plans = [BC.bsgs_plan({k: v * k_lvl for k, v in m.items()}, slots)
                          for m in cts]
        # EvalMod leaves sin(2π u) ≈ 2π c/q0; SlotToCoeff multiplies by V P, and the
        # factor sigma = q0 / (2π scale_0) is taken by the tracked scale (scale/sigma)
        self.sigma = self.q0 / (2.0 * math.pi * ch.scale_at[0])
        self.stc_plans = [BC.bsgs_plan(m, slots) for m in stc]
        self.cheb = BC.cheb_coeffs(BC.evalmod_function(K, r), degree)
        self._pt_cache: dict = {}
        self.conj = 2 * n - 1

    def _galois(self, step: int) -> int:
        return pow(5, step % self.slots, 2 * self.be.n)

    def _q(self, level: int) -> float:
        return float(self.be.chain.entry_products[level])

    # -- tracked-scale arithmetic --------------------------------------------------
    def _drop_to(self, x, level: int, scale: float):
        """Bring x down to `level` landing exactly on `scale` (restrict, integer
        factor, rescale: the reference's adjust trick with tracked scales)."""
        data, lvl, sc = x
        if lvl == level:
            return x
        be, ch = self.be, self.be.chain
        staging = level + 1
        ms = be._limbs(staging)
        factor = int(round(scale * self._q(staging) / sc))
        src = data if ms == data.shape[-2] else data[..., :ms, :].contiguous()
        y = ch.scalar_mul(src, ch.scalar_pairs(factor, range(ms)), ms)
        out = be._rescale_data(y, staging)
        return out, level, sc * factor / self._q(staging)

    def _align(self, a, b):
        if a[1] > b[1]:
            a = self._drop_to(a, b[1], b[2])
        elif b[1] > a[1]:
            b = self._drop_to(b, a[1], a[2])
        return a, b

    def _add(self, a, b, sub=False):
        a, b = self._align(a, b)
        if abs(a[2] - b[2]) > 2.0**-40 * abs(a[2]):
            raise RuntimeError(f"adding ciphertexts with scales {a[2]} != {b[2]} at level {a[1]}")
        m = self.be._limbs(a[1])
        f = self.be.chain.sub if sub else self.be.chain.add
        return f(a[0], b[0], m), a[1], a[2]

    def _mul(self, a, b):
        a, b = self._align(a, b)
        out = self.be._hmult(a[0].contiguous(), b[0].contiguous(), a[1])
        return out, a[1] - 1, a[2] * b[2] / self._q(a[1])

    def _mul_const(self, a, c: float, out_scale: float = None):
        """c * a, one level; lands exactly on out_scale (default: a's scale)."""
        data, lvl, sc = a
        q = self._q(lvl)
        pt_scale = q if out_scale is None else out_scale * q / sc
        pt = self._const_pt(c, lvl, pt_scale)
        m = self.be._limbs(lvl)
        out = self.be._rescale_data(self.be.chain.mul(data, pt, m, b_rows=m), lvl)
        return out, lvl - 1, sc * pt_scale / q

    def _const_pt(self, c: float, lvl: int, scale: float):
        """NTT-form plaintext of the constant slot vector c at `scale`: part of
        the bootstrapping constants, kept in this object's cache (like the
        BSGS diagonals) rather than the backend's per-step encode cache."""
        key = ("const", float(c), lvl, float(scale))
        pt = self._pt_cache.get(key)
        if pt is None:
            pt = self._pt_cache[key] = self.be._encode_rns(
                np.full(self.slots, c), lvl, ntt=True, scale=scale, limit=2.0**62)
        return pt

    def _restrict(self, a, level: int):
        """Drop limbs down to `level` (exact; the scale is unchanged)."""
        data, lvl, sc = a
        if lvl == level:
            return a
        assert lvl > level
        return data[..., : self.be._limbs(level), :].contiguous(), level, sc

    def _add_const(self, a, c: float):
        """(c0 + pt, c1) for every item: the plaintext pair [pt, 0] broadcast."""
        data, lvl, sc = a
        m = self.be._limbs(lvl)
        key = ("const2", float(c), lvl, float(sc))
        pt2 = self._pt_cache.get(key)
        if pt2 is None:
            pt = self._const_pt(c, lvl, sc)
            pt2 = torch.zeros(2, m, self.be.n, dtype=pt.dtype, device=pt.device)
            pt2[0].copy_(pt)
            pt2 = self._pt_cache[key] = self.be.chain.publish(pt2)
        out = self.be.chain.ew(0, torch.empty_like(data), data, pt2, limbs=m, b_rows=2 * m)
        return out, lvl, sc

    def _double(self, a):
        return self.be.chain.add(a[0], a[0], self.be._limbs(a[1])), a[1], a[2]

    # -- linear transforms ------------------------------------------------------------
    def _linear(self, x, plan, tag, out_scale: float = None):
        """sum_g rot(sum_b pt_gb * rot(x, b s), g n1 s), hoisted baby steps.  The
        diagonals are encoded at q_level (scale preserved) or so that the result
        lands on out_scale."""
        be, ch = self.be, self.be.chain
        data, lvl, sc = x
        s, n1, rows = plan
        m = be._limbs(lvl)
        q = self._q(lvl)
        pt_scale = q if out_scale is None else out_scale * q / sc
        babies = sorted({b for row in rows.values() for b in row if b})
        small = data.reshape(-1, 2, m, be.n).shape[0] <= self.stream_batch_max
        stack = (be.hoisted_rotations(data, lvl, [self._galois(b * s) for b in babies],
                                      stack=True, streams=self._side if small else None)
                 if babies else None)
        slot = {b: i for i, b in enumerate(babies)}
        slot[0] = -1  # the unrotated input
        data = data.contiguous().view(-1, 2, m, be.n)
        bsz, k = data.shape[0], ch.k
        # giant rows are independent up to the final sum: small batches spread
        # them over side streams (CUDA-graph branches when captured) so the
        # rows' kernels, each too small to fill the GPU, run side by side;
        # every stream keeps its own partial sums, added on the caller's stream
        ns = self.streams if bsz <= self.stream_batch_max else 0
        main = torch.cuda.current_stream()
        parts = []  # (acc, addend) per stream
        for st in self._side[:ns]:
            st.wait_stream(main)
        for gi, (g, row) in enumerate(sorted(rows.items())):
            if ns:
                si = gi % ns
                while len(parts) <= si:
                    parts.append([None, None])
                acc, addend = parts[si]
                ctx = torch.cuda.stream(self._side[si])
            else:
                if not parts:
                    parts.append([None, None])
                acc, addend = parts[0]
                ctx = contextlib.nullcontext()
            with ctx:
                acc, addend = self._giant_row(data, stack, slot, tag, g, row, lvl, pt_scale,
                                              n1, s, m, k, bsz, acc, addend)
            parts[si if ns else 0] = [acc, addend]
        if ns:
            for st in self._side[:ns]:
                main.wait_stream(st)
            for a, d in parts:
                for t in (a, d):
                    if t is not None:
                        t.record_stream(main)
        acc, addend = parts[0]
        for a, d in parts[1:]:
            if a is not None:
                acc = a if acc is None else ch.add(acc, a, m + k, out=acc, lmap=ch.ext_map(m))
            if d is not None:
                addend = d if addend is None else ch.add(addend, d, m, out=addend)
        e = len(ch.entry_primes[lvl])
        if acc is None:
            out = be._rescale_data(addend, lvl)
        else:
            tail = addend[:, :, m - e:m].reshape(2 * bsz, e, be.n)
            out = ch.divround_ntt(acc, 2 * bsz, m + k, k, e, addend=addend, addend_polys=2,
                                  addend_period=2, addend_stride=2, addend_tail=tail,
                                  basis=ch.ext_basis(m))
            out = out.view(bsz, 2, m - e, be.n)
        return out.view(*x[0].shape[:-2], m - e, be.n), lvl - 1, sc * pt_scale / q

    def _giant_row(self, data, stack, slot, tag, g, row, lvl, pt_scale, n1, s, m, k, bsz,
                   acc, addend):
        """One giant row of a BSGS transform added into (acc [Q u P], addend [Q])."""
        be, ch = self.be, self.be.chain
        if True:
            # one multiply-accumulate pass over the row's terms (ckb_pt_mac)
            key = (tag, g, lvl, pt_scale)
            hit = self._pt_cache.get(key)
            if hit is None:
                pts = torch.stack([be.encode_complex_ntt(diag, lvl, scale=pt_scale)
                                   for diag in row.values()])
                hit = self._pt_cache[key] = (ch.publish(pts), [slot[b] for b in row])
            pts, idx = hit
            inner = torch.empty_like(data)
            for lo in range(0, len(idx), 64):
                part = ch.pt_mac(data, stack, idx[lo:lo + 64], pts[lo:lo + 64], m,
                                 out=inner if lo == 0 else None)
                if lo:
                    ch.add(inner, part, m, out=inner)
            if not g:
                addend = inner if addend is None else ch.add(addend, inner, m, out=addend)
                return acc, addend
            # giant step: the rotation's key switch is accumulated in the
            # extended basis Q u P (rotation commutes with the exact rescale),
            # its c0' joins the addend; one ModDown + rescale ends the level
            galois = self._galois(g * n1 * s)
            r = ch.automorphism_ntt(inner, galois)
            c1 = ch.ntt_from(r[:, 1], bsz, m, 2 * m * be.n, inverse=True)
            ks = be._key_switch_acc(c1, m, batch=bsz, key=be.rotation_key(galois), own=r[:, 1],
                                    own_stride=2 * m * be.n)
            acc = ks if acc is None else ch.add(acc, ks, m + k, out=acc, lmap=ch.ext_map(m))
            # only c0' joins the addend: clear c1' (the key switch has read it)
            # and add the whole item (contiguous rows)
            r[:, 1].zero_()
            addend = r if addend is None else ch.add(addend, r, m, out=addend)
            return acc, addend

    # -- EvalMod ------------------------------------------------------------------
    def _chebyshev_basis(self, x):
        """T_1..T_16, T_32, T_64 (T_2j = 2 T_j^2 - 1, T_2j+1 = 2 T_j T_j+1 - T_1),
        computed depth by depth: the products of one depth are independent, so
        for small batches they go to the side streams (as _linear's giant rows)."""
        T = {1: x}

        def one(k):
            if k % 2 == 0:
                h = T[k // 2]
                return self._add_const(self._double(self._mul(h, h)), -1.0)
            a, b = T[k // 2], T[k // 2 + 1]
            return self._add(self._double(self._mul(a, b)), T[1], sub=True)

        main = torch.cuda.current_stream()
        par = x[0].shape[0] <= 2 * self.stream_batch_max
        for grp in ([2], [3, 4], [5, 6, 7, 8], list(range(9, 17)), [32], [64]):
            if not par or len(grp) == 1:
                for k in grp:
                    T[k] = one(k)
                continue
            side = self._side
            for st in side:
                st.wait_stream(main)
            for i, k in enumerate(grp):
                with torch.cuda.stream(side[i % len(side)]):
                    T[k] = one(k)
            for st in side:
                main.wait_stream(st)
            for k in grp:
                T[k][0].record_stream(main)
        return T

    def _eval_cheb(self, c, T, level: int, scale: float, par: bool = False):
        """sum_k c_k T_k as a ciphertext exactly at (level, scale): every term
        is steered onto the target by the scale of its coefficient plaintext
        (leaves) or of its quotient (giant-step products), so same-level
        additions never mix scales."""
        c = np.asarray(c, dtype=np.float64)
        deg = len(c) - 1
        while deg > 0 and c[deg] == 0.0:
            deg -= 1
        c = c[: deg + 1]
        if deg < 16:
            # leaf: sum_k c_k T_k at (level + 1, scale * q) in one pass — a
            # constant slot vector encodes to the integer round(c * pt_scale),
            # so every term is an integer multiple of T_k read at level + 1
            # (ckb_scalar_mac) — then a single rescale onto (level, scale)
            be, ch = self.be, self.be.chain
            lvl = level + 1
            m = be._limbs(lvl)
            q = self._q(lvl)
            ks = [k for k in range(1, deg + 1) if c[k] != 0.0] or [1]
            key = ("leaf", c.tobytes(), level, float(scale),
                   tuple((T[k][1], float(T[k][2])) for k in ks))
            sc = self._pt_cache.get(key)
            if sc is None:
                for k in ks:
                    assert T[k][1] >= lvl, "Chebyshev leaf below its operands' level"
                ints = [int(np.rint(c[k] * (scale * q / T[k][2]))) for k in ks]
                sc = self._pt_cache[key] = ch.scalar_table(ints, m)
            acc = ch.scalar_mac([T[k][0].contiguous() for k in ks], sc, m)
            acc = be._rescale_data(acc, lvl)
            return self._add_const((acc, level, scale), c[0])
        n = 1 << (deg.bit_length() - 1)
        q = np.zeros(deg - n + 1)
        q[0] = c[n]
        q[1:] = 2.0 * c[n + 1:]
        rem = c[:n].copy()
        for j in range(1, deg - n + 1):
            rem[n - j] -= c[n + j]
        tn = self._restrict(T[n], level + 1)
        qscale = scale * self._q(level + 1) / tn[2]
        if not par:
            qv = self._eval_cheb(q, T, level + 1, qscale)
            prod = self._mul(qv, tn)
            return self._add(prod, self._eval_cheb(rem, T, level, scale))
        # par: the quotient and remainder subtrees are independent — one side
        # stream each (small batches), joined for the giant-step product
        main = torch.cuda.current_stream()
        sq, sr = self._side[0], self._side[1]
        sq.wait_stream(main)
        sr.wait_stream(main)
        with torch.cuda.stream(sq):
            prod = self._mul(self._eval_cheb(q, T, level + 1, qscale), tn)
        with torch.cuda.stream(sr):
            rv = self._eval_cheb(rem, T, level, scale)
        main.wait_stream(sq)
        main.wait_stream(sr)
        prod[0].record_stream(main)
        rv[0].record_stream(main)
        return self._add(prod, rv)

    def _cheb_level(self, T, deg: int) -> int:
        """Lowest-depth target level: leaves need T_1..T_15 one level above."""
        leaf = min(T[k][1] for k in range(1, 16)) - 1
        splits = max(0, deg.bit_length() - 4)  # giant steps 16, 32, 64, ...
        return leaf - splits

    def _evalmod(self, x):
        T = self._chebyshev_basis(x)
        y = self._eval_cheb(self.cheb, T, self._cheb_level(T, len(self.cheb) - 1), x[2],
                            par=x[0].shape[0] <= 2 * self.stream_batch_max)
        for _ in range(self.r):
            y = self._add_const(self._double(self._mul(y, y)), -1.0)
        return y

    # -- the whole procedure ----------------------------------------------------------
    def bootstrap(self, ct: GpuCiphertext) -> GpuCiphertext:
        """ct.data [2, m, N] or a batch [B, 2, m, N] (all at ct.level)."""
        be, ch = self.be, self.be.chain
        single = ct.data.dim() == 3
        if single:
            ct = GpuCiphertext(ct.data.unsqueeze(0), ct.level)
        raised = be.mod_raise(ct)
        x = (raised.data, raised.level, float(self.q0))  # read at scale q0: slots = V u'
        for t, plan in enumerate(self.cts_plans):
            x = self._linear(x, plan, ("cts", t))
        data, lvl, sc = x
        m = be._limbs(lvl)
        conj = be.rotate_data(data, lvl, self.conj)
        re = ch.add(data, conj, m)
        mono = be.monomial_ntt(3 * be.n // 2, lvl)  # -X^{N/2}: multiplies slots by -i
        im = ch.mul(ch.sub(data, conj, m), mono, m, b_rows=m)
        # the real and imaginary parts through one batched EvalMod (same level
        # and scale; every op is per-ciphertext, so results are unchanged)
        bsz = data.shape[0]
        y, l_y, s_y = self._evalmod((torch.cat([re, im]), lvl, sc))
        y_re = (y[:bsz], l_y, s_y)
        y_im = (ch.mul(y[bsz:].contiguous(), be.monomial_ntt(be.n // 2, l_y), be._limbs(l_y),
                       b_rows=be._limbs(l_y)), l_y, s_y)
        z = self._add(y_re, y_im)
        z = (z[0], z[1], z[2] / self.sigma)
        rl = be.params.refresh_level
        for t, plan in enumerate(self.stc_plans):
            last = t == len(self.stc_plans) - 1
            target = ch.scale_at[z[1] - 1] if last else None
            z = self._linear(z, plan, ("stc", t), out_scale=target)
        data, lvl, sc = z
        if lvl > rl:
            data, lvl, sc = self._drop_to(z, rl, ch.scale_at[rl])
        if lvl < rl:
            raise RuntimeError(f"bootstrapping consumed too many levels ({lvl} < {rl})")
        return GpuCiphertext(data[0] if single else data, lvl)
