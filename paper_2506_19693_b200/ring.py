"""Device-resident RNS chain and thin wrappers over the sm_100a kernels.

``GpuChain`` plays the role of the reference's ``ChainContext``
(ckks/ring.py:21-59): the prime chain ordered [base | rescale entries | special],
level -> limb-prefix map, the scale schedule, plus the device tables the
kernels read (twiddles, Barrett/Shoup constants, pairwise inverses).

Polynomials are torch.uint64 CUDA tensors ``[..., limbs, N]`` (contiguous,
canonical residues); the prime of limb i at level l is ``all_primes[i]`` for
the ciphertext prefix and ``all_primes[LQ + t]`` for special prime t, so the
kernels' per-limb prime index is simply the position in ``all_primes``.
Every wrapper launches on the caller's current CUDA stream.
"""

from __future__ import annotations

import math
import os

import numpy as np
import torch

from . import _native as nat
from .primes import build_chain

U64 = torch.uint64
W = 8  # bytes per residue


def shoup(v: int, p: int) -> int:
    return (v << 64) // p


class KernelTimer:
    """Optional per-kernel CUDA-event timing (bench.py): every wrapper call
    records start/end events on the launching (current) stream plus its
    algorithmic bytes and kernel-launch count."""

    def __init__(self):
        self.records = []

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for name, s, e, nbytes, launches, f64_bytes in self.records:
            d = out.setdefault(name, {"ms": 0.0, "calls": 0, "bytes": 0, "launches": 0,
                                      "f64_bytes": 0})
            d["ms"] += s.elapsed_time(e)
            d["calls"] += 1
            d["bytes"] += nbytes
            d["launches"] += launches
            d["f64_bytes"] += f64_bytes
        return out


TIMER = None  # set to a KernelTimer to instrument


def _run(name, nbytes, launches, fn, f64_share=None):
    """f64_share: callable giving the fraction of the work on the FP64 NTT path
    (rows whose prime is < 2^46), evaluated only when instrumenting."""
    t = TIMER
    if t is None:
        return fn()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    r = fn()
    e.record()
    t.records.append((name, s, e, nbytes, launches,
                      nbytes * f64_share() if f64_share is not None else 0))
    return r


class GpuChain:
    # ModUp and the fast-conversion ModDown correction on the tensor cores
    # (csrc/tc.cu, CKB_RING_TC; bit-identical to the CUDA-core kernels, which
    # CKB_NO_TC=1 selects for A/B runs).  Per chain: set_ring_flag(RING_TC, ...).
    use_tc = os.environ.get("CKB_NO_TC") != "1"

    def __init__(self, params, layout: str = "reference", device=None):
        self.params = params
        self.layout = layout
        self.n = params.poly_degree
        self.log_n = self.n.bit_length() - 1
        self.device = torch.device(device or "cuda")
        entries, scale_at = build_chain(params, layout)
        self.entry_primes = entries
        self.special_primes = list(entries[-1])
        self.primes = [p for e in entries[:-1] for p in e]
        self.all_primes = self.primes + self.special_primes
        self.lq = len(self.primes)
        self.k = len(self.special_primes)
        self.level_limbs = [len(entries[0])]
        for e in entries[1:-1]:
            self.level_limbs.append(self.level_limbs[-1] + len(e))
        self.entry_products = [math.prod(e) for e in entries]
        self.special_product = math.prod(self.special_primes)
        self.scale_at = scale_at
        mods, ntt, pair = nat.build_tables(self.log_n, self.all_primes)
        dev = self.device
        self._mods = torch.from_numpy(mods).to(dev)
        self._ntt = torch.from_numpy(ntt.reshape(-1)).to(dev)
        self._pair = torch.from_numpy(pair.reshape(-1)).to(dev)
        self.ring = nat.CkbRing(self.log_n, len(self.all_primes), self._mods.data_ptr(),
                                self._ntt.data_ptr(), self._pair.data_ptr(),
                                (nat.ctypes.c_uint64 * 2)(*nat.f64_mask(self.all_primes)))
        self.ring.wide_mask = (nat.ctypes.c_uint64 * 2)(*nat.wide_mask(self.all_primes))
        self.ring.mid_mask = (nat.ctypes.c_uint64 * 2)(*nat.mid_mask(self.all_primes))
        if self.use_tc:  # outputs of the basis conversions only feed forward NTTs
            self.ring.flags |= nat.RING_TC | nat.RING_LAZY_BCONV
        self.ring_p = nat.ctypes.pointer(self.ring)
        self._maps: dict = {}

    def set_ntt_chunk_bytes(self, nbytes: int) -> int:
        """L2 budget of this chain's two-phase transforms (ckb_ring.ntt_chunk_bytes,
        0 = the 96 MB default); returns the previous value.  The struct is ours:
        the library reads it at every call and keeps no state."""
        prev = int(self.ring.ntt_chunk_bytes)
        self.ring.ntt_chunk_bytes = int(nbytes)
        return prev

    def set_ring_flag(self, flag: int, on: bool) -> bool:
        """Set / clear a ckb_ring.flags bit (nat.RING_*); returns the previous state."""
        prev = bool(self.ring.flags & flag)
        self.ring.flags = (self.ring.flags | flag) if on else (self.ring.flags & ~flag)
        return prev

    # -- bases ------------------------------------------------------------------
    # A basis is a tuple of indices into all_primes; the kernels receive it as
    # a ctypes int32 array (cached per tuple).
    def limbs_at(self, level: int) -> list:
        return self.primes[: self.level_limbs[level]]

    def modulus_at(self, level: int) -> int:
        return math.prod(self.limbs_at(level))

    def q_basis(self, m: int) -> tuple:
        """The first m ciphertext limbs."""
        return tuple(range(m))

    def ext_basis(self, m: int, k: int = None) -> tuple:
        """Ciphertext limbs [0, m) followed by the (first k) special primes
        (keys.py:81)."""
        k = self.k if k is None else k
        return tuple(range(m)) + tuple(range(self.lq, self.lq + k))

    def all_basis(self) -> tuple:
        return tuple(range(len(self.all_primes)))

    def cmap(self, basis: tuple):
        hit = self._maps.get(basis)
        if hit is None:
            hit = self._maps[basis] = nat.i32_array(basis)
        return hit

    # legacy helpers (ctypes maps)
    def q_map(self, m: int):
        return self.cmap(self.q_basis(m))

    def ext_map(self, m: int, k: int = None):
        return self.cmap(self.ext_basis(m, k))

    def all_map(self):
        return self.cmap(self.all_basis())

    def custom_map(self, idx: tuple):
        return self.cmap(tuple(idx))

    def scalar_pairs(self, value: int, primes_idx) -> object:
        """{v mod p, shoup} pairs for ckb_scalar_mul / ckb_divround prescale."""
        vals = []
        for i in primes_idx:
            p = self.all_primes[i]
            v = value % p
            vals += [v, shoup(v, p)]
        return nat.u64_array(vals)

    def publish(self, t: torch.Tensor) -> torch.Tensor:
        """A lazily built, cached device table computed ON THE DEVICE: wait once
        for it to be complete so groups issued on other streams (executor
        fork/join, bootstrap side streams) can read it.  Host-built tables go
        through upload_table instead, which does not drain the queue."""
        if t is not None and t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        return t

    _upload_stream = None

    def upload_table(self, arr: np.ndarray) -> torch.Tensor:
        """Host-built constant table -> device, complete on return, WITHOUT
        waiting for the compute work queued on the current stream: staged in
        pinned memory and copied on a private side stream, whose copy alone the
        host waits for (a pageable .to(device) or a current-stream sync would
        drain the GPU's queue at every first use of a table: ~1.4 s of idle GPU
        in a config-5 step).  Complete before any later launch on any stream."""
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if self.device.type != "cuda":
            return t.to(self.device)
        if GpuChain._upload_stream is None:
            GpuChain._upload_stream = torch.cuda.Stream(device=self.device)
        st = GpuChain._upload_stream
        pinned = t.pin_memory()
        with torch.cuda.stream(st):
            out = pinned.to(self.device, non_blocking=True)
        st.synchronize()
        return out

    def _drop_chain_table(self, basis: tuple, n_drop: int) -> torch.Tensor:
        """Mixed-radix constants for dropping the last n_drop limbs of basis
        (see ckb_divround): per limb j, {M_u mod p_j} for u < n_drop then
        {M_t^-1 mod p_j} (t = j's drop position, n_drop for kept limbs)."""
        primes = [self.all_primes[i] for i in basis]
        limbs = len(primes)
        drops = [primes[limbs - 1 - u] for u in range(n_drop)]
        tab = np.zeros((limbs, n_drop + 1, 2), dtype=np.uint64)
        for j, p in enumerate(primes):
            pos = limbs - 1 - j
            t = pos if pos < n_drop else n_drop
            prod = 1
            for u in range(n_drop):
                if u < t:
                    c = prod % p
                    tab[j, u] = (c, shoup(c, p))
                prod *= drops[u]
            mt = math.prod(drops[:t]) % p
            inv = pow(mt, -1, p)
            tab[j, n_drop] = (inv, shoup(inv, p))
        return self.upload_table(tab.reshape(-1))

    def drop_tables(self, basis: tuple, n1: int, n2: int):
        key = ("drop", basis, n1, n2)
        hit = self._maps.get(key)
        if hit is None:
            t1 = self._drop_chain_table(basis, n1) if n1 else None
            t2 = self._drop_chain_table(basis[: len(basis) - n1], n2) if n2 else None
            hit = self._maps[key] = (t1, t2)
        return hit

    # -- allocation ---------------------------------------------------------------
    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(*shape, self.n, dtype=U64, device=self.device)

    # -- kernels -------------------------------------------------------------------
    def _ntt_launches(self, rows: int) -> int:
        """Kernel launches of one transform call: one per phase and L2 chunk
        (a launch holding both prime classes is one per-CTA-dispatch kernel)."""
        if self.log_n <= 12:
            return 1
        budget = self.ring.ntt_chunk_bytes or nat.DEFAULT_NTT_CHUNK_BYTES
        chunk = max(1, int(budget) // (self.n * W))
        return 2 * (-(-rows // chunk))

    F64_PRIME_LIMIT = nat.F64_PRIME_LIMIT
    use_hps = True  # wide ModDown drops via the fast basis-conversion correction
    fuse_combine = True  # ModDown combine as the E transform's epilogue

    def _f64_share(self, lmap, limbs: int):
        return lambda: sum(self.all_primes[lmap[i]] < self.F64_PRIME_LIMIT
                           for i in range(limbs)) / limbs

    def ntt_fwd(self, t: torch.Tensor, limbs: int, lmap=None):
        rows = t.numel() >> self.log_n
        lm = lmap or self.q_map(limbs)
        _run("ntt", 2 * rows * self.n * W, self._ntt_launches(rows), lambda: nat.check(
            nat.LIB.ckb_ntt_forward(self.ring_p, nat.ptr(t), rows, limbs, lm,
                                    nat.stream_handle()),
            "ntt_forward"), self._f64_share(lm, limbs))
        return t

    def ntt_inv(self, t: torch.Tensor, limbs: int, lmap=None):
        rows = t.numel() >> self.log_n
        lm = lmap or self.q_map(limbs)
        _run("intt", 2 * rows * self.n * W, self._ntt_launches(rows), lambda: nat.check(
            nat.LIB.ckb_ntt_inverse(self.ring_p, nat.ptr(t), rows, limbs, lm,
                                    nat.stream_handle()),
            "ntt_inverse"), self._f64_share(lm, limbs))
        return t

    def ntt_from(self, src: torch.Tensor, items: int, limbs: int, item_stride: int,
                 inverse: bool = False, lmap=None, out=None):
        """Out-of-place (i)NTT of `items` items of [limbs][N] read at
        src + i*item_stride elements (a strided view, e.g. one component of a
        [B, 3, limbs, N] tensor) into a fresh contiguous [items, limbs, N]."""
        out = out if out is not None else torch.empty(items, limbs, self.n, dtype=U64,
                                                      device=self.device)
        rows = items * limbs
        lm = lmap or self.q_map(limbs)
        fn = nat.LIB.ckb_ntt_inverse_from if inverse else nat.LIB.ckb_ntt_forward_from
        _run("intt" if inverse else "ntt", 2 * rows * self.n * W, self._ntt_launches(rows),
             lambda: nat.check(fn(self.ring_p, nat.ptr(out), nat.ptr(src), item_stride, rows,
                                  limbs, lm, nat.stream_handle()), "ntt_from"),
             self._f64_share(lm, limbs))
        return out

    def ew(self, op: int, out, a, b=None, c=None, limbs: int = 0, lmap=None, b_rows: int = 0):
        rows = a.numel() >> self.log_n
        nb = 2 * rows + (0 if b is None else (b_rows or rows)) + (0 if c is None else rows)
        _run("elementwise", nb * self.n * W, 1, lambda: nat.check(nat.LIB.ckb_elementwise(
            self.ring_p, op, nat.ptr(out), nat.ptr(a), nat.ptr(b) if b is not None else None,
            nat.ptr(c) if c is not None else None, rows, limbs, lmap or self.q_map(limbs), b_rows,
            nat.stream_handle()), "elementwise"))
        return out

    def pt_mac(self, x0, stack, term_idx, pts, limbs: int, out=None, lmap=None):
        """sum_t X_t (.) pts[t] (ckb_pt_mac): X_t = x0 for term_idx[t] == -1, else
        stack[term_idx[t]]; every X_t shaped like x0 ([..., limbs, N]); pts
        [T, limbs, N] broadcast over the leading rows."""
        ref = x0 if x0 is not None else stack[0]
        out = out if out is not None else torch.empty_like(ref)
        rows = ref.numel() >> self.log_n
        t = len(term_idx)
        sst = stack[0].numel() if stack is not None else 0
        nb = t * rows + t * limbs + rows
        _run("pt_mac", nb * self.n * W, 1, lambda: nat.check(nat.LIB.ckb_pt_mac(
            self.ring_p, nat.ptr(out), nat.ptr(x0) if x0 is not None else None,
            nat.ptr(stack) if stack is not None else None, sst, nat.i32_array(term_idx),
            nat.ptr(pts), limbs * self.n, t, rows, limbs, lmap or self.q_map(limbs),
            nat.stream_handle()), "pt_mac"))
        return out

    def scalar_table(self, scalars, limbs: int) -> torch.Tensor:
        """Device [K][limbs] residues of Python-int scalars (any sign) for
        scalar_mac; build once and reuse (no upload inside graph captures)."""
        tab = np.array([[int(a) % self.all_primes[j] for j in range(limbs)] for a in scalars],
                       dtype=np.uint64)
        return self.upload_table(tab.reshape(-1))

    def scalar_mac(self, terms, sc: torch.Tensor, limbs: int, out=None):
        """sum_k a_k * terms[k] (ckb_scalar_mac): terms are ciphertext tensors
        [..., m_k, N] with m_k >= limbs (read restricted to the first `limbs`),
        the same leading shape; sc = scalar_table([a_k], limbs)."""
        lead = terms[0].shape[:-2]
        polys = int(np.prod(lead)) if len(lead) else 1
        if any(t.shape[:-2] != lead or not t.is_contiguous() for t in terms):
            raise ValueError("scalar_mac terms must be contiguous with one leading shape")
        out = out if out is not None else torch.empty(*lead, limbs, self.n, dtype=U64,
                                                      device=self.device)
        ptrs = (nat.c_vp * len(terms))(*[t.data_ptr() for t in terms])
        tl = nat.i32_array([t.shape[-2] for t in terms])
        nb = len(terms) * polys * limbs + polys * limbs
        _run("scalar_mac", nb * self.n * W, 1, lambda: nat.check(nat.LIB.ckb_scalar_mac(
            self.ring_p, nat.ptr(out), ptrs, tl, nat.ptr(sc), len(terms), polys, limbs,
            self.q_map(limbs), nat.stream_handle()), "scalar_mac"))
        return out

    def add(self, a, b, limbs, out=None, lmap=None):
        return self.ew(0, out if out is not None else torch.empty_like(a), a, b, limbs=limbs, lmap=lmap)

    def sub(self, a, b, limbs, out=None, lmap=None):
        return self.ew(1, out if out is not None else torch.empty_like(a), a, b, limbs=limbs, lmap=lmap)

    def mul(self, a, b, limbs, out=None, lmap=None, b_rows=0):
        return self.ew(2, out if out is not None else torch.empty_like(a), a, b, limbs=limbs,
                       lmap=lmap, b_rows=b_rows)

    def neg(self, a, limbs, out=None, lmap=None):
        return self.ew(3, out if out is not None else torch.empty_like(a), a, limbs=limbs, lmap=lmap)

    def scalar_mul(self, a, pairs, limbs, out=None, lmap=None):
        out = out if out is not None else torch.empty_like(a)
        rows = a.numel() >> self.log_n
        _run("scalar_mul", 2 * rows * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_scalar_mul(self.ring_p, nat.ptr(out), nat.ptr(a), rows, limbs,
                                   lmap or self.q_map(limbs), pairs, nat.stream_handle()),
            "scalar_mul"))
        return out

    def tensor(self, a, b, limbs, out=None):
        batch = a.numel() // (2 * limbs * self.n)
        out = out if out is not None else torch.empty(batch, 3, limbs, self.n, dtype=U64,
                                                      device=self.device)
        _run("tensor", 7 * batch * limbs * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_tensor(self.ring_p, nat.ptr(out), nat.ptr(a), nat.ptr(b), batch, limbs,
                               self.q_map(limbs), nat.stream_handle()), "tensor"))
        return out

    def modup(self, d, m: int, alpha: int, bconv, batch: int = None, in_batch_stride: int = 0,
              skip_own: bool = False, out=None, k: int = None):
        """d: batch items of [m][N] (item b at d + b*in_batch_stride elements).
        Returns digits [batch, rows, N]: nd * ext rows, or with skip_own the
        compact layout without each digit's own limbs (len(digit_basis(...)) rows;
        a short last digit keeps ext - width rows)."""
        if batch is None:
            batch = d.numel() // (m * self.n)
        k = self.k if k is None else k
        ext = m + k
        rows = len(self.digit_basis(m, alpha, True, k)) if skip_own else -(-m // alpha) * ext
        out = out if out is not None else torch.empty(batch, rows, self.n, dtype=U64,
                                                      device=self.device)
        _run("modup", (batch * m + batch * rows) * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_modup(self.ring_p, nat.ptr(out), nat.ptr(d), in_batch_stride, batch,
                              m, self.q_map(m), ext, self.ext_map(m, k), alpha,
                              nat.ptr(bconv) if bconv is not None else None, int(skip_own),
                              nat.stream_handle()), "modup"))
        return out

    def digit_basis(self, m: int, alpha: int, skip_own: bool, k: int = None) -> tuple:
        """Per-row prime indices of a digits tensor [nd][rows] (for its NTT)."""
        ext = self.ext_basis(m, k)
        if not skip_own:
            return ext
        nd = -(-m // alpha)
        out = ()
        for j in range(nd):
            own = set(range(j * alpha, min((j + 1) * alpha, m)))
            out += tuple(pi for e, pi in enumerate(ext) if e not in own)
        return out

    def fold_table(self, m: int, k: int) -> torch.Tensor:
        """[m][2] {P_k mod q_e, shoup}: the special modulus of a k-prime key switch
        on the first m Q limbs (ckb_ks_inner_fold)."""
        key = ("fold", m, k)
        hit = self._maps.get(key)
        if hit is None:
            pk = math.prod(self.special_primes[:k])
            vals = []
            for q in self.primes[:m]:
                v = pk % q
                vals += [v, shoup(v, q)]
            hit = self._maps[key] = self.upload_table(np.array(vals, dtype=np.uint64))
        return hit

    def ks_inner(self, digits, m: int, alpha: int = 1, key: torch.Tensor = None,
                 key_ptrs: torch.Tensor = None, own: torch.Tensor = None, own_bstride: int = 0,
                 out=None, k: int = None, fold=None):
        """digits: ckb_modup's output ([batch, rows, N]; skip_own layout when own
        is given).  fold = (b, b_stride, a, a_stride): addends (tensors or views
        with item stride *_stride elements; a may be None) folded into the Q limbs
        as addend * P, so the ModDown that follows yields x P^-1 + addend."""
        batch = digits.shape[0]
        nd = -(-m // alpha)
        k = self.k if k is None else k
        ext = m + k
        out = out if out is not None else torch.empty(batch, 2, ext, self.n, dtype=U64,
                                                      device=self.device)
        key_limbs = self.lq + k  # keys over Q u (first k special primes)
        n_keys = batch if key_ptrs is not None else 1
        nb = batch * nd * ext + n_keys * nd * 2 * ext + batch * 2 * ext  # own rows counted as read
        if fold is None:
            _run("ks_inner", nb * self.n * W, 1, lambda: nat.check(
                nat.LIB.ckb_ks_inner(self.ring_p, nat.ptr(out), nat.ptr(digits), batch, nd, ext,
                                     self.ext_map(m, k), alpha, m,
                                     nat.ptr(own) if own is not None else None, own_bstride,
                                     nat.ptr(key) if key is not None else None,
                                     nat.ptr(key_ptrs) if key_ptrs is not None else None,
                                     key_limbs, self.ext_map(m, k), nat.stream_handle()),
                "ks_inner"))
            return out
        fb, fbs, fa, fas = fold
        nb += batch * m * (1 if fa is None else 2)
        ftab = self.fold_table(m, k)
        _run("ks_inner", nb * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_ks_inner_fold(self.ring_p, nat.ptr(out), nat.ptr(digits), batch, nd, ext,
                                      self.ext_map(m, k), alpha, m,
                                      nat.ptr(own) if own is not None else None, own_bstride,
                                      nat.ptr(key) if key is not None else None,
                                      nat.ptr(key_ptrs) if key_ptrs is not None else None,
                                      key_limbs, self.ext_map(m, k), nat.ptr(fb), fbs,
                                      nat.ptr(fa) if fa is not None else None, fas,
                                      nat.ptr(ftab), m, nat.stream_handle()), "ks_inner_fold"))
        return out

    # digits' row-phase NTT fused with the key inner product (ckb_ks_ntt_mac,
    # N = 2^16 / 2^17).  Bit-identical to the unfused path (tests) but slower
    # on the config-2 batch (6.0 ms vs 4.7 ms for NTT + ks_inner per 64-ct
    # HMult: three serial row passes per CTA at 16 warps/SM), so off by default.
    fuse_ks_mac = False

    def ks_ntt_mac(self, digits, m: int, alpha: int, key: torch.Tensor = None,
                   key_ptrs: torch.Tensor = None, own: torch.Tensor = None, own_bstride: int = 0,
                   out=None, k: int = None):
        """Forward NTT of ckb_modup's skip_own digits fused with the inner
        product (ckb_ks_ntt_mac): acc [batch, 2, m + k, N], NTT domain; the
        digits tensor is scratch afterwards."""
        batch = digits.shape[0]
        nd = -(-m // alpha)
        k = self.k if k is None else k
        ext = m + k
        out = out if out is not None else torch.empty(batch, 2, ext, self.n, dtype=U64,
                                                      device=self.device)
        basis = self.digit_basis(m, alpha, True, k)
        rows = batch * len(basis)
        n_keys = batch if key_ptrs is not None else 1
        nb = 2 * rows + n_keys * nd * 2 * ext + batch * (m + 2 * ext)  # NTT r/w, keys, own, acc
        _run("ks_ntt_mac", nb * self.n * W, self._ntt_launches(rows), lambda: nat.check(
            nat.LIB.ckb_ks_ntt_mac(self.ring_p, nat.ptr(out), nat.ptr(digits), batch, m, alpha,
                                   ext, self.ext_map(m, k), self.cmap(basis), nat.ptr(own),
                                   own_bstride,
                                   nat.ptr(key) if key is not None else None,
                                   nat.ptr(key_ptrs) if key_ptrs is not None else None,
                                   self.lq + k, self.ext_map(m, k), nat.stream_handle()),
            "ks_ntt_mac"), self._f64_share(self.cmap(basis), len(basis)))
        return out

    def divround(self, x, polys: int, limbs: int, n1: int, n2: int = 0, addend=None,
                 addend_polys: int = 0, addend_period: int = 1, addend_stride: int = None,
                 prescale=None, in_poly_stride: int = 0, basis: tuple = None, out=None):
        basis = basis if basis is not None else self.q_basis(limbs)
        m2 = limbs - n1 - n2
        out = out if out is not None else torch.empty(polys, m2, self.n, dtype=U64,
                                                      device=self.device)
        if addend_stride is None:
            addend_stride = addend_polys
        t1, t2 = self.drop_tables(basis, n1, n2)
        n_add = 0 if addend is None else (polys // addend_period) * addend_polys * (limbs - n1)
        nb = polys * limbs + n_add + polys * m2
        _run("divround", nb * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_divround(self.ring_p, nat.ptr(out), nat.ptr(x), in_poly_stride,
                                 nat.ptr(addend) if addend is not None else None,
                                 addend_polys if addend is not None else 0,
                                 addend_period, addend_stride, polys, limbs, self.cmap(basis),
                                 n1, n2, prescale, nat.ptr(t1) if t1 is not None else None,
                                 nat.ptr(t2) if t2 is not None else None, nat.stream_handle()),
            "divround"))
        return out

    def _corr_table(self, basis: tuple, n1: int, n2: int) -> torch.Tensor:
        """tabE for ckb_divround_ntt_corr: per output limb j, {M1_u * P1^-1 mod q_j}
        for u < n1, {M2_u mod q_j} for u < n2, then {C_j, 0} with C_j the smallest
        multiple of q_j >= 2^59 (shifts the signed remainders, |r| < 2^59, to [0, 2^61))."""
        primes = [self.all_primes[i] for i in basis]
        limbs = len(primes)
        m1 = limbs - n1
        m2 = m1 - n2
        d1 = [primes[limbs - 1 - u] for u in range(n1)]
        d2 = [primes[m1 - 1 - u] for u in range(n2)]
        P1 = math.prod(d1)
        tab = np.zeros((m2, n1 + n2 + 1, 2), dtype=np.uint64)
        for j in range(m2):
            p = primes[j]
            tab[j, n1 + n2] = (p * -(-(1 << 59) // p), 0)  # C_j: multiple of q_j in [2^59, 2^61)
            p1inv = pow(P1 % p, -1, p)
            for u in range(n1):
                c = math.prod(d1[:u]) % p * p1inv % p
                tab[j, u] = (c, shoup(c, p))
            for u in range(n2):
                c = math.prod(d2[:u]) % p
                tab[j, n1 + u] = (c, shoup(c, p))
        return self.upload_table(tab.reshape(-1))

    HPS_MIN_DROP = 6  # csrc/ops.cu kHpsMinDrop

    def _hps_table(self, basis: tuple, n1: int) -> torch.Tensor:
        """tabH for ckb_divround_ntt_corr: per kept limb j < m1, {p_u^-1 mod q_j}
        for the dropped primes p_u (u = 0 the last limb), then per dropped prime
        {(P1/p_u)^-1 mod p_u, shoup}."""
        primes = [self.all_primes[i] for i in basis]
        limbs = len(primes)
        m1 = limbs - n1
        d1 = [primes[limbs - 1 - u] for u in range(n1)]
        P1 = math.prod(d1)
        tab = np.zeros(m1 * n1 + 2 * n1, dtype=np.uint64)
        for j in range(m1):
            q = primes[j]
            for u, p in enumerate(d1):
                tab[j * n1 + u] = pow(p % q, -1, q)
        for u, p in enumerate(d1):
            w = pow((P1 // p) % p, -1, p)
            tab[m1 * n1 + 2 * u] = w
            tab[m1 * n1 + 2 * u + 1] = shoup(w, p)
        return self.upload_table(tab)

    def hps_table(self, basis: tuple, n1: int, n2: int):
        if n1 < self.HPS_MIN_DROP or n2 > 2:
            return None
        key = ("hps", basis, n1)
        hit = self._maps.get(key)
        if hit is None:
            hit = self._maps[key] = self._hps_table(basis, n1)
        return hit

    def corr_table(self, basis: tuple, n1: int, n2: int) -> torch.Tensor:
        key = ("corr", basis, n1, n2)
        hit = self._maps.get(key)
        if hit is None:
            hit = self._maps[key] = self._corr_table(basis, n1, n2)
        return hit

    def divround_ntt(self, x, polys: int, limbs: int, n1: int, n2: int = 0, *,
                     x_poly_stride: int = 0, addend=None, addend_polys: int = 0,
                     addend_period: int = 1, addend_stride: int = None, addend_tail=None,
                     basis: tuple = None, out=None, post=None):
        """Exact divide-and-round of NTT-domain polys (see ckb_divround_ntt_corr):
        iNTT of the dropped limbs, correction polynomial, its NTT, combine.
        post: [polys, m2, N] NTT-domain polys added to the result in the same
        pass (ckb_divround_ntt_combine_acc; the s + rotate(s) accumulate).
        addend_tail: [polys, n2, N] NTT-domain copy of the addend's limbs
        [limbs-n1-n2, limbs-n1) (zeros for polys without an addend) when n2 > 0."""
        basis = basis if basis is not None else self.q_basis(limbs)
        n = self.n
        m1 = limbs - n1
        m2 = m1 - n2
        xs = x_poly_stride if x_poly_stride else limbs * n
        if addend_stride is None:
            addend_stride = addend_polys
        has_add = addend is not None and n2 > 0
        trows = n1 + n2 + (n2 if has_add else 0)
        tbasis = tuple(basis[m2:]) + (tuple(basis[m2:m1]) if has_add else ())
        xv = x.as_strided((polys, n1 + n2, n), (xs, n, 1), x.storage_offset() + m2 * n)
        if has_add:
            T = torch.empty(polys, trows, n, dtype=U64, device=self.device)
            T[:, : n1 + n2].copy_(xv)
            T[:, n1 + n2:].copy_(addend_tail)
            self.ntt_inv(T, trows, self.cmap(tbasis))
        else:  # the dropped limbs transformed straight out of x (no staging copy)
            T = self.ntt_from(xv, polys, trows, xs, inverse=True, lmap=self.cmap(tbasis))
        t1, t2 = self.drop_tables(basis, n1, n2)
        tE = self.corr_table(basis, n1, n2)
        tH = self.hps_table(basis, n1, n2) if self.use_hps else None
        E = torch.empty(polys, m2, n, dtype=U64, device=self.device)
        nb = polys * trows + polys * m2
        _run("divround_corr", nb * n * W, 1, lambda: nat.check(
            nat.LIB.ckb_divround_ntt_corr(self.ring_p, nat.ptr(E), nat.ptr(T), int(has_add), polys,
                                          limbs, self.cmap(basis), n1, n2,
                                          nat.ptr(t1) if t1 is not None else None,
                                          nat.ptr(t2) if t2 is not None else None, nat.ptr(tE),
                                          nat.ptr(tH) if tH is not None else None,
                                          nat.stream_handle()), "divround_ntt_corr"))
        out = out if out is not None else torch.empty(polys, m2, n, dtype=U64, device=self.device)
        n_add = 0 if addend is None else (polys // addend_period) * addend_polys * m2
        if post is not None and (post.dtype != U64 or not post.is_contiguous()
                                 or post.numel() != polys * m2 * n):
            raise ValueError("post must be contiguous uint64 [polys, m2, N]")
        args = (nat.ptr(x), xs, nat.ptr(addend) if addend is not None else None,
                addend_polys if addend is not None else 0, addend_period, addend_stride)
        tabs = (nat.ptr(t1) if t1 is not None else None, nat.ptr(t2) if t2 is not None else None,
                nat.ptr(post) if post is not None else None, 0, nat.stream_handle())
        if self.fuse_combine:
            # E's forward NTT with the combine as its last phase's store (E in,
            # out written; the transformed E never goes back to HBM)
            nb = polys * m2 * (3 if post is None else 4) + n_add  # E read + x, out
            _run("ntt_combine", nb * n * W, self._ntt_launches(polys * m2), lambda: nat.check(
                nat.LIB.ckb_ntt_forward_combine(self.ring_p, nat.ptr(out), nat.ptr(E), *args,
                                                polys, limbs, self.cmap(basis), n1, n2, *tabs),
                "ntt_forward_combine"), self._f64_share(self.cmap(tuple(basis[:m2])), m2))
            return out
        self.ntt_fwd(E, m2, self.cmap(tuple(basis[:m2])))
        nb = polys * m2 * (3 if post is None else 4) + n_add
        _run("divround_combine", nb * n * W, 1, lambda: nat.check(
            nat.LIB.ckb_divround_ntt_combine_acc(
                self.ring_p, nat.ptr(out), *args, nat.ptr(E), polys, limbs, self.cmap(basis),
                n1, n2, *tabs), "divround_ntt_combine"))
        return out

    def automorphism_ntt(self, x, galois: int, out=None, g_items=None, rows_per_item: int = 0):
        out = out if out is not None else torch.empty_like(x)
        rows = x.numel() >> self.log_n
        _run("automorphism", 2 * rows * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_automorphism_ntt(self.ring_p, nat.ptr(out), nat.ptr(x), rows, galois,
                                         nat.ptr(g_items) if g_items is not None else None,
                                         rows_per_item, nat.stream_handle()),
            "automorphism_ntt"))
        return out

    def automorphism(self, x, galois: int, limbs: int, out=None, lmap=None, ginv_items=None,
                     rows_per_item: int = 0):
        """X -> X^galois per row; with ginv_items (device u64 [items]) each item of
        rows_per_item rows uses its own galois^-1 mod 2N."""
        out = out if out is not None else torch.empty_like(x)
        rows = x.numel() >> self.log_n
        _run("automorphism", 2 * rows * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_automorphism(self.ring_p, nat.ptr(out), nat.ptr(x), rows, limbs,
                                     lmap or self.q_map(limbs), galois,
                                     nat.ptr(ginv_items) if ginv_items is not None else None,
                                     rows_per_item, nat.stream_handle()), "automorphism"))
        return out

    def reduce(self, x: torch.Tensor, limbs: int, out=None, lmap=None):
        """x mod p per limb for arbitrary 64-bit words (after an all-reduce)."""
        out = out if out is not None else torch.empty_like(x)
        rows = x.numel() >> self.log_n
        _run("reduce", 2 * rows * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_reduce(self.ring_p, nat.ptr(out), nat.ptr(x), rows, limbs,
                               lmap or self.q_map(limbs), nat.stream_handle()), "reduce"))
        return out

    def sample(self, seeds: torch.Tensor, limbs: int, uniform: bool = True, gaussian: bool = True,
               sigma: float = 3.2, lmap=None):
        """Device samples per item: uniform residues [items, limbs, N] and
        rounded Gaussian int64 [items, N] (ckb_sample)."""
        items = seeds.numel()
        a = torch.empty(items, limbs, self.n, dtype=U64, device=self.device) if uniform else None
        e = torch.empty(items, self.n, dtype=torch.int64, device=self.device) if gaussian else None
        _run("sample", items * (limbs + 1) * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_sample(self.ring_p, nat.ptr(a) if a is not None else None,
                               nat.ptr(e) if e is not None else None, nat.ptr(seeds), items, limbs,
                               lmap or self.q_map(limbs), sigma, nat.stream_handle()), "sample"))
        return a, e

    def from_i64(self, coeffs: torch.Tensor, limbs: int, lmap=None, out=None):
        polys = coeffs.numel() >> self.log_n
        out = out if out is not None else torch.empty(polys, limbs, self.n, dtype=U64,
                                                      device=self.device)
        _run("from_i64", (polys + polys * limbs) * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_from_i64(self.ring_p, nat.ptr(out), nat.ptr(coeffs), polys, limbs,
                                 lmap or self.q_map(limbs), nat.stream_handle()), "from_i64"))
        return out

    def to_f64(self, x: torch.Tensor, limbs: int, lmap=None):
        polys = x.numel() // (limbs * self.n)
        out = torch.empty(polys, self.n, dtype=torch.float64, device=self.device)
        _run("to_f64", (polys * limbs + polys) * self.n * W, 1, lambda: nat.check(
            nat.LIB.ckb_to_f64(self.ring_p, nat.ptr(out), nat.ptr(x), polys, limbs,
                               lmap or self.q_map(limbs), nat.stream_handle()), "to_f64"))
        return out

    # -- host <-> device helpers -------------------------------------------------------
    def packed_bytes(self, items: int, limbs: int, lmap=None) -> int:
        """Size of the packed transfer format (ckb_pack) of [items][limbs][N]."""
        return int(nat.LIB.ckb_packed_bytes(self.ring_p, items, limbs, lmap or self.q_map(limbs)))

    def pack(self, x: torch.Tensor, items: int, limbs: int, lmap=None, out=None) -> torch.Tensor:
        """[items][limbs][N] residues -> uint8 packed transfer format (5 bytes per
        residue below 2^40, 6 below 2^48, else 8): fewer PCIe bytes per copy."""
        lm = lmap or self.q_map(limbs)
        nb = self.packed_bytes(items, limbs, lm)
        out = out if out is not None else torch.empty(nb, dtype=torch.uint8, device=self.device)
        _run("pack", items * limbs * self.n * W + nb, 1, lambda: nat.check(
            nat.LIB.ckb_pack(self.ring_p, nat.ptr(out), nat.ptr(x), items, limbs, lm,
                             nat.stream_handle()), "pack"))
        return out

    def unpack(self, packed: torch.Tensor, items: int, limbs: int, lmap=None,
               out=None) -> torch.Tensor:
        """Inverse of pack: -> [items, limbs, N] uint64."""
        lm = lmap or self.q_map(limbs)
        out = out if out is not None else torch.empty(items, limbs, self.n, dtype=U64,
                                                      device=self.device)
        _run("unpack", items * limbs * self.n * W + packed.numel(), 1, lambda: nat.check(
            nat.LIB.ckb_unpack(self.ring_p, nat.ptr(out), nat.ptr(packed), items, limbs, lm,
                               nat.stream_handle()), "unpack"))
        return out

    def upload_u64(self, arr: np.ndarray) -> torch.Tensor:
        return self.upload_table(np.ascontiguousarray(arr, dtype=np.uint64))
