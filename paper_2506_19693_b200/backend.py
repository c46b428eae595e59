"""B200 RNS-CKKS backend: the drop-in for the reference's ``CkksBackend``.

Boundary (/root/reference/pkg/src/ciphermlp/api.py:129-259): a ``Backend``
subclass with ``backend_id = "ckks"`` implementing the five payload hooks
(_payload_elementwise / _rotate / _encrypt / _decrypt / _bootstrap) plus
serialize_cipher / deserialize_cipher, constructor-compatible with
``CkksBackend(params, rotation_indices=(), rng_seed=0, bootstrap_eps=0.0,
keyset_id=None, _secret=None)`` (ckks/backend.py:55-75).  Level, depth and
keyset checks stay in the shared base class.

Payload: ``GpuCiphertext(data, level)`` — ``data`` is a torch.uint64 CUDA
tensor [2, limbs(level), N] holding (c0, c1) in the NTT (evaluation) domain.
The reference keeps ciphertexts in the coefficient domain (backend.py:1-9);
here they rest in the evaluation domain so multiplies need no forward
transforms, and the divide-and-round steps (ModDown, rescale) are applied as
NTT-domain corrections — the same integers, so ``planes_of`` (one inverse
NTT) is bit-identical to the reference's planes.  Every integer operation
runs in the sm_100a kernels (ring.py -> _native.py -> libckks_b200.so); the
host does only what the reference's host does besides arithmetic: numpy
sampling with the reference's RNG streams (so keys and encryptions are
reproducible bit-for-bit against it), the float-64 encode/decode FFT (cuFFT via
torch on the device), error checks and serialisation.

Extra keyword options (all default to the reference's behaviour):
  prime_layout  "reference" | "baseline" | "schedule"   (primes.py)
  dnum          None = per-limb digits (reference, keys.py:84-97); an int gives
                hybrid key switching with digits of ceil(LQ/dnum) limbs
  secret_hw     None = dense ternary (ring.py:161-162); h = ternary with exactly
                h non-zeros (BASELINE configs: 64 / 192)
  device        CUDA device (default: current)
  encoder       "device" (cuFFT) | "numpy" (the reference's host FFT, bit-identical
                encodings/decodings: mode-A whole-step parity tests only)
  deferred      record HE calls and run them batched (executor.WaveExecutor) when a
                result is decrypted / serialized / flushed (deferred.py)
"""

from __future__ import annotations

import collections
import contextlib
import dataclasses
import io
import json
import math
import numbers
import struct

import numpy as np
import torch

from . import he_api, he_errors
from .ring import U64, GpuChain, shoup

CT_MAGIC = b"RBCT"
KEY_MAGIC = b"RBKY"
SERIAL_VERSION = 1
ERROR_SIGMA = 3.2
MAX_SAFE_COEFF = float(2**52)


# While a CUDA graph is being captured (graphs.GraphedStep), the pinned
# staging tensors of in-graph uploads are kept alive here for the graph's life,
# as (tag, pinned tensor) pairs: a replay reads whatever the pinned tensor then
# holds, so GraphedStep rewrites the encryption-seed uploads ("seeds", serials)
# before every replay (fresh randomness per replayed step).
H2D_KEEPALIVE = None


def _h2d(arr: np.ndarray, device, tag=None) -> torch.Tensor:
    """Host array -> device without a stream sync: staged through pinned memory
    (torch's caching host allocator) and copied asynchronously.  A plain copy
    from pageable memory would make the host wait for all queued GPU work."""
    t = torch.from_numpy(np.array(arr, copy=True, order="C"))  # writable, owned
    if torch.device(device).type != "cuda":
        return t.to(device)
    pinned = t.pin_memory()
    if H2D_KEEPALIVE is not None:
        H2D_KEEPALIVE.append((tag, pinned))
    return pinned.to(device, non_blocking=True)


@dataclasses.dataclass(frozen=True)
class GpuCiphertext:
    """(c0, c1) at one chain level; NTT domain (bit-reversed evaluation slots of
    NttPlan.forward), canonical residues."""

    data: torch.Tensor  # [2, limbs, N] uint64, CUDA
    level: int

    @property
    def c0(self):
        return self.data[0]

    @property
    def c1(self):
        return self.data[1]


class DeviceEncoder:
    """Canonical embedding with the rotation-friendly 5^i slot order
    (encoding.py:17-76), evaluated with cuFFT in float64 on the device.

    host=True (backend option encoder="numpy", for mode-A whole-step bit
    identity only): the float64 FFTs run with numpy on the host exactly as
    encoding.py:34-54 writes them, so encodings and decodings round like the
    reference's (cuFFT and pocketfft differ in the last ulp, which moves a
    rint by one in ~1 coefficient per encode).  The integer work around it
    (residues, NTT, the CRT lift) stays on the device."""

    def __init__(self, n: int, device, host: bool = False):
        self.n = n
        self.device = device
        self.host = bool(host)
        slots = n // 2
        exps = np.empty(slots, dtype=np.int64)
        e = 1
        for i in range(slots):
            exps[i] = e
            e = e * 5 % (2 * n)
        self.bins_np = (exps - 1) // 2
        self.conj_bins_np = (2 * n - exps - 1) // 2
        self.bins = torch.from_numpy(self.bins_np).to(device)
        self.conj_bins = torch.from_numpy(self.conj_bins_np).to(device)
        twist = np.exp(1j * np.pi * np.arange(n) / n)
        self.twist_np = twist
        self.untwist_np = np.conj(twist)
        self.twist = torch.from_numpy(twist).to(device)
        self.untwist = torch.from_numpy(np.conj(twist)).to(device)
        self.bins32 = torch.from_numpy(
            np.concatenate([self.bins_np, self.conj_bins_np]).astype(np.int32)).to(device)

    def embed_residues(self, values: np.ndarray, scale: float, chain, limbs: int,
                       need_max: bool = False):
        """[B, <= N/2] real slot rows -> residues [B, limbs, N] of their encodings
        (encoding.py:34-49 + ring.py:139-145): ckb_embed_scatter, cuFFT,
        ckb_embed_finish (twist, rint and every limb's residue in one pass).
        need_max: also the exact max |coefficient| (a device scalar) for the
        overflow checks the host-side bound could not clear."""
        from . import _native as nat

        vals = np.ascontiguousarray(np.atleast_2d(np.asarray(values, dtype=np.float64)))
        b, w = vals.shape
        n = self.n
        v = _h2d(vals, self.device) if w else torch.zeros(b, 1, dtype=torch.float64,
                                                          device=self.device)
        spec = torch.empty(b, n, dtype=torch.complex128, device=self.device)
        nat.check(nat.LIB.ckb_embed_scatter(nat.ptr(spec), nat.ptr(v), b, w, w, float(scale),
                                            nat.ptr(self.bins32), n.bit_length() - 1,
                                            nat.stream_handle()), "embed_scatter")
        spec = torch.fft.fft(spec, dim=1)
        res = torch.empty(b, limbs, n, dtype=torch.uint64, device=self.device)
        mx = torch.zeros(1, dtype=torch.int64, device=self.device) if need_max else None
        nat.check(nat.LIB.ckb_embed_finish(chain.ring_p, nat.ptr(res), nat.ptr(spec), b, limbs,
                                           chain.q_map(limbs), nat.ptr(self.twist),
                                           nat.ptr(mx) if mx is not None else None,
                                           nat.stream_handle()), "embed_finish")
        return res, mx

    def _embed_host(self, rows: np.ndarray, scale: float) -> torch.Tensor:
        """encoding.py:34-49 per row (numpy), -> rounded float64 on the device."""
        out = np.empty((rows.shape[0], self.n))
        for i, vals in enumerate(rows):
            v = np.zeros(self.n // 2)
            v[: vals.shape[0]] = vals
            spectrum = np.zeros(self.n, dtype=np.complex128)
            scaled = v * scale
            spectrum[self.bins_np] = scaled
            spectrum[self.conj_bins_np] = scaled
            w = np.fft.fft(spectrum) / self.n
            out[i] = np.rint(np.real(w * self.untwist_np))
        return _h2d(out, self.device)

    def embed_device(self, values, scale: float) -> torch.Tensor:
        """Real slots -> int64 coefficients [N] on the device (encoding.py:34-49)."""
        if self.host:
            return self._embed_host(np.asarray(values, dtype=np.float64)[None], scale)[0]
        v = _h2d(np.asarray(values, dtype=np.float64), self.device)
        spec = torch.zeros(self.n, dtype=torch.complex128, device=self.device)
        scaled = torch.zeros(self.n // 2, dtype=torch.float64, device=self.device)
        scaled[: v.shape[0]] = v * scale
        spec[self.bins] = scaled.to(torch.complex128)
        spec[self.conj_bins] = scaled.to(torch.complex128)
        w = torch.fft.fft(spec) / self.n
        return torch.round(torch.real(w * self.untwist))

    def embed_device_batch(self, values: np.ndarray, scale: float) -> torch.Tensor:
        """[B, <= N/2] real slot rows -> [B, N] coefficients (one batched FFT)."""
        if self.host:
            return self._embed_host(np.asarray(values, dtype=np.float64), scale)
        v = _h2d(np.asarray(values, dtype=np.float64), self.device)
        b = v.shape[0]
        spec = torch.zeros(b, self.n, dtype=torch.complex128, device=self.device)
        scaled = torch.zeros(b, self.n // 2, dtype=torch.float64, device=self.device)
        scaled[:, : v.shape[1]] = v * scale
        sc = scaled.to(torch.complex128)
        spec[:, self.bins] = sc
        spec[:, self.conj_bins] = sc
        w = torch.fft.fft(spec, dim=1) / self.n
        return torch.round(torch.real(w * self.untwist))

    def embed_complex_device(self, z, scale: float) -> torch.Tensor:
        """Complex slots -> int64 coefficients (conjugate spectrum on the mirrored bins)."""
        zt = torch.as_tensor(np.asarray(z, dtype=np.complex128), device=self.device) * scale
        spec = torch.zeros(self.n, dtype=torch.complex128, device=self.device)
        spec[self.bins[: zt.shape[0]]] = zt
        spec[self.conj_bins[: zt.shape[0]]] = torch.conj(zt)
        w = torch.fft.fft(spec) / self.n
        return torch.round(torch.real(w * self.untwist))

    def embed(self, values, scale: float) -> np.ndarray:
        coeffs = self.embed_device(values, scale)
        if float(coeffs.abs().max()) >= MAX_SAFE_COEFF:
            raise he_errors.EncodingOverflow(
                "scaled values exceed the exactly-representable coefficient range")
        return coeffs.to(torch.int64).cpu().numpy()

    def unembed_device(self, coeffs: torch.Tensor, scale: float) -> torch.Tensor:
        if self.host:  # encoding.py:51-55 per row (numpy)
            c = coeffs.cpu().numpy()
            rows = c.reshape(-1, self.n)
            out = np.empty((rows.shape[0], self.n // 2))
            for i, r in enumerate(rows):
                spectrum = np.fft.ifft(r.astype(np.float64) * self.twist_np) * self.n
                out[i] = np.real(spectrum[self.bins_np]) / scale
            return torch.from_numpy(out.reshape(*c.shape[:-1], self.n // 2))
        w = coeffs.to(torch.complex128) * self.twist
        spec = torch.fft.ifft(w) * self.n
        return torch.real(spec[..., self.bins]) / scale

    def unembed(self, coeffs, scale: float) -> np.ndarray:
        c = torch.as_tensor(np.asarray(coeffs, dtype=np.float64), device=self.device)
        return self.unembed_device(c, scale).cpu().numpy()


class SecretKey:
    """Holds the ternary secret (``coeffs``, as ring.py:161-162 / keys.py:37-46)
    and its NTT form over every prime (``s_full``, [all_limbs, N])."""

    def __init__(self, coeffs: np.ndarray, s_full: torch.Tensor):
        self.coeffs = coeffs
        self.s_full = s_full


@dataclasses.dataclass
class KeySwitchKey:
    """Rows [digits][2 (b, a)][all limbs][N] uint64, NTT domain (keys.py:29-34)."""

    data: torch.Tensor


class B200CkksCore:
    """Payload hooks; mixed into a ``Backend`` base (ours or the reference's)."""

    backend_id = "ckks"
    _errors = he_errors
    _api = he_api
    _instances = 0
    # ModDown addends (HMult's d0/d1, HRot's c0') folded into the key inner
    # product as addend * P (ckb_ks_inner_fold) instead of read by the ModDown
    # correction and combine; same integers.  CKB_NO_FOLD=1 for A/B runs.
    fold_addends = __import__("os").environ.get("CKB_NO_FOLD") != "1"

    def __init__(self, params, rotation_indices=(), rng_seed: int = 0, bootstrap_eps: float = 0.0,
                 keyset_id=None, _secret=None, *, prime_layout: str = "reference", dnum=None,
                 secret_hw=None, device=None, encode_cache: int = 512,
                 conjugation_key: bool = False, real_bootstrap: bool = False,
                 sampler: str = None, low_special=None, encoder: str = "device",
                 deferred: bool = False, deferred_max_group: int = None,
                 deferred_async: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 CKKS backend needs a CUDA device; there is no CPU path")
        if keyset_id is None:
            B200CkksCore._instances += 1
            keyset_id = f"b200-keyset-{B200CkksCore._instances}"
        super().__init__(params, keyset_id)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.chain = GpuChain(params, prime_layout, self.device)
        self.ctx = self.chain
        ch = self.chain
        self.n = params.poly_degree
        if encoder not in ("device", "numpy"):
            raise self._errors.InvalidParameters(f"unknown encoder {encoder!r}")
        self.encoder = DeviceEncoder(self.n, self.device, host=encoder == "numpy")
        self.rng_seed = rng_seed
        self.bootstrap_eps = bootstrap_eps
        # "numpy": the reference's default_rng streams (bit-exact keys/encryptions,
        # ring.py:148-162, backend.py:174); "philox": counter-based device
        # sampling (ckb_sample), one stream per (seed, serial) — the default
        # off the reference prime layout, where no bit-exact stream exists.
        self.sampler = sampler or ("numpy" if prime_layout == "reference" else "philox")
        if self.sampler not in ("numpy", "philox"):
            raise self._errors.InvalidParameters(f"unknown sampler {self.sampler!r}")
        self._ksk_count = 0
        self.rotation_indices = frozenset(int(k) for k in rotation_indices)
        self.real_bootstrap = bool(real_bootstrap)
        key_steps = set(self.rotation_indices)
        if self.real_bootstrap:
            if prime_layout != "bootstrap" or not params.bootstrap_depth:
                raise self._errors.InvalidParameters(
                    "real_bootstrap needs prime_layout='bootstrap' and bootstrap_depth > 0")
            from .bootstrap import bootstrap_rotations

            key_steps |= bootstrap_rotations(params)
            conjugation_key = True
        self._bootstrapper = None
        self.alpha = 1 if dnum is None else max(1, -(-ch.lq // int(dnum)))
        self.dnum = dnum
        self._bconv_cache: dict = {}
        self._adjust_cache: dict = {}
        self._enc_cache: collections.OrderedDict = collections.OrderedDict()
        self._enc_cache_cap = encode_cache
        # the reference's 2^52 exactness guard (encoding.py:46-48); the bootstrap
        # layout encodes top-level values at ~2^60 where float64 rounding
        # (2^-52 relative) is far below the noise
        self._encode_limit = float(2**62) if prime_layout == "bootstrap" else MAX_SAFE_COEFF
        rng = np.random.default_rng(rng_seed)
        coeffs = rng.integers(-1, 2, self.n).astype(np.int64)  # ring.py:161-162
        if secret_hw is not None:
            coeffs = _hw_secret(self.n, int(secret_hw), rng_seed)
        if _secret is not None:
            coeffs = np.asarray(_secret).astype(np.int64)
        self.sk = SecretKey(coeffs, self._to_ntt_all(coeffs))
        self.relin_key = self._make_ksk(self._mul_all(self.sk.s_full, self.sk.s_full), rng)
        self.galois_for_step: dict = {}
        self.rotation_keys: dict = {}
        slots = params.slot_count
        s_coeff = ch.ntt_inv(self.sk.s_full.clone(), len(ch.all_primes), ch.all_map())
        for step in sorted({k % slots for k in key_steps} - {0}):
            g = pow(5, step, 2 * self.n)
            self.galois_for_step[step] = g
            s_rot = ch.automorphism(s_coeff, g, len(ch.all_primes), lmap=ch.all_map())
            ch.ntt_fwd(s_rot, len(ch.all_primes), ch.all_map())
            self.rotation_keys[g] = self._make_ksk(s_rot, rng)
        if conjugation_key:  # X -> X^(2N-1): complex conjugation of the slots
            g = 2 * self.n - 1
            s_rot = ch.automorphism(s_coeff, g, len(ch.all_primes), lmap=ch.all_map())
            ch.ntt_fwd(s_rot, len(ch.all_primes), ch.all_map())
            self.rotation_keys[g] = self._make_ksk(s_rot, rng)
        # Level-aware special modulus: a ciphertext at level l key-switches over
        # Q u P' with P' the first k(l) special primes, P' above the widest
        # digit at l (the key-switch noise then stays ~N*sigma, far below the
        # scale), so the ModUp / inner product / ModDown of the training steps'
        # multiplies and rotations carry fewer 60-bit limbs.  low_special: an
        # int k' (levels <= refresh level) or tiers [(max_level, k), ...]; own
        # relin and rotation keys (user steps) per k.  Bootstrapping always
        # uses the full P (its precision budget assumes 2^120 of headroom).
        # Off by default (the parity tests pin the full-P semantics).
        self.k_low = None
        self._ks_tiers = []
        self._force_full_p = False
        self.relin_keys_k: dict = {}
        self.rotation_keys_k: dict = {}
        if isinstance(low_special, str):
            if low_special != "auto":
                raise self._errors.InvalidParameters(f"unknown low_special {low_special!r}")
            low_special = self._auto_tiers() or None
        if low_special is not None:
            if isinstance(low_special, numbers.Integral):
                tiers = [(params.refresh_level, int(low_special))]
            else:
                try:
                    tiers = sorted((int(l), int(k)) for l, k in low_special)
                except (TypeError, ValueError):
                    raise self._errors.InvalidParameters(
                        "low_special: an int or [(max_level, k), ...]") from None
            for max_level, kk in tiers:
                if not 0 < kk < ch.k:
                    raise self._errors.InvalidParameters(
                        f"low_special: {kk} special primes for levels <= {max_level}; need "
                        f"0 < k' < {ch.k}")
                if not 0 <= max_level <= params.level:
                    raise self._errors.InvalidParameters(
                        f"low_special: tier level {max_level} outside 0..{params.level}")
                m = ch.level_limbs[min(max_level, params.level)]
                widest = max(math.prod(ch.all_primes[lo:min(lo + self.alpha, m)])
                             for lo in range(0, m, self.alpha))
                if math.prod(ch.special_primes[:kk]) <= widest:
                    raise self._errors.InvalidParameters(
                        f"low_special: {kk} special primes do not cover a digit at level "
                        f"{max_level} ({widest.bit_length()} bits)")
                self._ks_tiers.append((max_level, kk))
                if kk in self.relin_keys_k:
                    continue
                self.relin_keys_k[kk] = self._make_ksk(
                    self._mul_all(self.sk.s_full, self.sk.s_full), rng, k=kk)
                rk = self.rotation_keys_k[kk] = {}
                for step in sorted({k % slots for k in self.rotation_indices} - {0}):
                    g = self.galois_for_step[step]
                    s_rot = ch.automorphism(s_coeff, g, len(ch.all_primes), lmap=ch.all_map())
                    ch.ntt_fwd(s_rot, len(ch.all_primes), ch.all_map())
                    rk[g] = self._make_ksk(s_rot, rng, k=kk)
            if self._ks_tiers:
                self.k_low = self._ks_tiers[0][1]
        self._bs_rng = np.random.default_rng(rng_seed + 0x5EED)
        # deferred=True: HE calls are recorded and run batched on the first
        # decrypt / serialize / flush (deferred.py)
        self._rec = None
        if deferred:
            from .deferred import Recorder

            self._rec = Recorder(self, max_group=deferred_max_group, pipelined=deferred_async)

    def flush(self, on_issued=None) -> None:
        """Run every deferred HE call recorded so far (no-op when eager).  With
        deferred_async the program is handed to the issuing thread and this
        returns at once; on_issued() runs right after its last launch."""
        if self._rec is not None:
            self._rec.flush(on_issued=on_issued)
        elif on_issued is not None:
            on_issued()

    def wait(self) -> None:
        """Join pipelined deferred programs (no-op otherwise)."""
        if self._rec is not None:
            self._rec.wait()

    # ------------------------------------------------------------------ keys
    AUTO_TIER_MARGIN_BITS = 0  # the same rule __init__ checks explicit tiers with

    def _auto_tiers(self) -> list:
        """low_special="auto": per level the fewest special primes whose product
        exceeds the widest digit at that level (times 2^AUTO_TIER_MARGIN_BITS;
        the key-switch error is then ~ sigma * sqrt(N) * digits, far below the
        ~2^45 scale), merged into tiers of consecutive levels; levels that need
        the whole P keep it.  Every tier costs its own relinearisation and
        rotation keys."""
        ch = self.chain
        need = []
        for lv in range(self.params.level + 1):
            m = ch.level_limbs[lv]
            widest = max(math.prod(ch.all_primes[lo:min(lo + self.alpha, m)])
                         for lo in range(0, m, self.alpha))
            target = widest << self.AUTO_TIER_MARGIN_BITS
            kk = next((k for k in range(1, ch.k + 1)
                       if math.prod(ch.special_primes[:k]) > target), ch.k)
            need.append(kk)
        tiers = []
        for lv, kk in enumerate(need):
            if kk >= ch.k:
                break  # levels above keep the full P
            if tiers and tiers[-1][1] == kk:
                tiers[-1] = (lv, kk)
            else:
                tiers.append((lv, kk))
        return tiers

    def _to_ntt_all(self, coeffs: np.ndarray) -> torch.Tensor:
        ch = self.chain
        t = torch.as_tensor(np.asarray(coeffs, dtype=np.int64), device=self.device)
        s = ch.from_i64(t, len(ch.all_primes), ch.all_map())[0]
        return ch.ntt_fwd(s, len(ch.all_primes), ch.all_map())

    def _mul_all(self, a, b):
        ch = self.chain
        return ch.mul(a, b, len(ch.all_primes), lmap=ch.all_map())

    def _make_ksk(self, source_ntt: torch.Tensor, rng, k: int = None) -> KeySwitchKey:
        """keys.py:49-71 on the device; row j holds P * source on the limbs of
        digit j (a single limb when alpha == 1, exactly the reference).  k: key
        over Q and the first k special primes only (P = their product)."""
        ch = self.chain
        k = ch.k if k is None else k
        full = ch.all_primes[: ch.lq + k]
        kl = len(full)
        amap = ch.cmap(tuple(range(kl)))
        special = math.prod(ch.special_primes[:k])
        rows = []
        digits = [(lo, min(lo + self.alpha, ch.lq)) for lo in range(0, ch.lq, self.alpha)]
        out = torch.empty(len(digits), 2, kl, self.n, dtype=U64, device=self.device)
        for j, (lo, hi) in enumerate(digits):
            if self.sampler == "philox":
                tag = 0x4B45590000 if k == ch.k else 0x4C4F570000  # low-P keys: own streams
                seed = torch.tensor([_mix64(self.rng_seed, tag + self._ksk_count, j)],
                                    dtype=torch.int64, device=self.device).view(U64)
                a_d, e_d = ch.sample(seed, kl, lmap=amap)
                a_np = None
            else:
                a_np = np.stack([rng.integers(0, p, self.n, dtype=np.uint64) for p in full])
                e_np = np.rint(rng.normal(0.0, ERROR_SIGMA, self.n)).astype(np.int64)
            if a_np is None:
                a = a_d[0]
                e = ch.from_i64(e_d, kl, amap)[0]
            else:
                a = ch.upload_u64(a_np)
                e = ch.from_i64(torch.from_numpy(e_np).to(self.device), kl, amap)[0]
            ch.ntt_fwd(e, kl, amap)
            b = ch.mul(a, self.sk.s_full[:kl].contiguous(), kl, lmap=amap)
            ch.sub(e, b, kl, out=b, lmap=amap)  # b = -a*s + e
            idx = tuple(range(lo, hi))
            lmap = ch.custom_map(idx)
            pv = ch.scalar_pairs(special, idx)
            msg = ch.scalar_mul(source_ntt[lo:hi].contiguous(), pv, hi - lo, lmap=lmap)
            b[lo:hi] = ch.add(b[lo:hi].contiguous(), msg, hi - lo, lmap=lmap)
            out[j, 0] = b
            out[j, 1] = a
            rows.append(j)
        self._ksk_count += 1
        return KeySwitchKey(out)

    def rotation_key(self, galois: int) -> KeySwitchKey:
        try:
            return self.rotation_keys[galois]
        except KeyError:
            raise self._errors.MissingRotationKey(f"no key for Galois element {galois}") from None

    # ------------------------------------------------------------------ helpers
    def _scale(self, level: int) -> float:
        return self.chain.scale_at[level]

    def _limbs(self, level: int) -> int:
        return self.chain.level_limbs[level]

    def _bconv(self, m: int, k: int = None):
        """ModUp tables for hybrid digits at a ciphertext with m limbs:
        [digit][i][ qhat_i^-1 mod q_i, shoup, ([qhat_i]_{p_e}, shoup) for e in ext ]."""
        if self.alpha == 1:
            return None
        ch = self.chain
        k = ch.k if k is None else k
        if (m, k) in self._bconv_cache:
            return self._bconv_cache[(m, k)]
        ext = list(range(m)) + list(range(ch.lq, ch.lq + k))
        nd = -(-m // self.alpha)
        width = 2 + 2 * len(ext)
        tab = np.zeros((nd, self.alpha, width), dtype=np.uint64)
        for j in range(nd):
            lo, hi = j * self.alpha, min((j + 1) * self.alpha, m)
            qs = ch.all_primes[lo:hi]
            Qj = math.prod(qs)
            for i, q in enumerate(qs):
                qhat = Qj // q
                inv = pow(qhat % q, -1, q)
                tab[j, i, 0] = inv
                tab[j, i, 1] = shoup(inv, q)
                for e, pi in enumerate(ext):
                    p = ch.all_primes[pi]
                    c = qhat % p
                    tab[j, i, 2 + 2 * e] = c
                    tab[j, i, 3 + 2 * e] = shoup(c, p)
        t = self.chain.upload_table(tab.reshape(-1))
        self._bconv_cache[(m, k)] = t
        return t

    def _key_switch_acc(self, d: torch.Tensor, m: int, batch: int = 1, d_stride: int = 0,
                        key: KeySwitchKey = None, key_ptrs=None, own: torch.Tensor = None,
                        own_stride: int = 0, k: int = None, fold=None) -> torch.Tensor:
        """keys.py:74-97: digits of d (coefficient domain, batch items of [m, N]
        at b*d_stride), lifted to Q_l u P, NTT, inner product with the key rows.
        ``own`` is the NTT form of d (items at b*own_stride): a digit's own
        limbs are then not re-transformed but read from it.  Returns the
        NTT-domain accumulator [batch, 2, m + k, N]; the division by P
        (keys.py:98-99) is left to the caller so it can fuse adds/rescales."""
        ch = self.chain
        a = self.alpha
        k = ch.k if k is None else k
        nd = -(-m // a)
        # own limbs read from the NTT-domain input (a short last digit included);
        # the digits' NTT limb map holds <= 128 rows
        skip = own is not None and nd * (m + k) - m <= 128
        digits = ch.modup(d, m, a, self._bconv(m, k), batch=batch, in_batch_stride=d_stride,
                          skip_own=skip, k=k)
        basis = ch.digit_basis(m, a, skip, k)
        if skip and ch.fuse_ks_mac and ch.log_n in (16, 17) and fold is None:
            # the digits' row-phase transform fused with the inner product
            return ch.ks_ntt_mac(digits, m, a, key=key.data if key is not None else None,
                                 key_ptrs=key_ptrs, own=own, own_bstride=own_stride, k=k)
        ch.ntt_fwd(digits, len(basis), ch.cmap(basis))
        return ch.ks_inner(digits, m, a, key=key.data if key is not None else None,
                           key_ptrs=key_ptrs, own=own if skip else None, own_bstride=own_stride,
                           k=k, fold=fold)

    def _can_fold(self, m: int) -> bool:
        """The ModDown addend can ride in the inner product (ckb_ks_inner_fold:
        hybrid digits, at most 8 of them; not the fused ks_ntt_mac path)."""
        return (self.fold_addends and self.alpha > 1 and -(-m // self.alpha) <= 8
                and not (self.chain.fuse_ks_mac and self.chain.log_n in (16, 17)))

    def _ks_k(self, level: int) -> int:
        """Special primes a key switch at this level uses (see __init__)."""
        if not self._force_full_p:
            for max_level, kk in self._ks_tiers:
                if level <= max_level:
                    return kk
        return self.chain.k

    def _low(self, level: int) -> bool:
        return self._ks_k(level) != self.chain.k

    def _adjust_to_level(self, ct: GpuCiphertext, target: int) -> GpuCiphertext:
        """backend.py:94-112: restrict to target+1 limbs, multiply by the integer
        that lands the target scale, rescale (NTT domain)."""
        if ct.level == target:
            return ct
        if ct.level < target:
            raise self._errors.IncompatibleOperands("cannot raise a ciphertext's level")
        return GpuCiphertext(self._adjust_data(ct.data, ct.level, target), target)

    def _adjust_data(self, data: torch.Tensor, origin: int, target: int) -> torch.Tensor:
        """_adjust_to_level on [..., 2, limbs(origin), N] (any batch shape)."""
        ch = self.chain
        staging = target + 1
        ms = self._limbs(staging)
        key = (origin, target)
        if key not in self._adjust_cache:
            s_star = self._scale(target) * ch.entry_products[staging] / self._scale(origin)
            factor = int(np.rint(s_star))
            self._adjust_cache[key] = ch.scalar_pairs(factor, range(ms))
        # out-of-place: payloads are immutable (api.py:51-65), never scale in place
        src = data if ms == data.shape[-2] else data[..., :ms, :].contiguous()
        x = ch.scalar_mul(src, self._adjust_cache[key], ms)
        polys = x.numel() // (ms * self.n)
        out = ch.divround_ntt(x, polys, ms, len(ch.entry_primes[staging]))
        return out.view(*data.shape[:-2], ms - len(ch.entry_primes[staging]), self.n)

    def _rescale(self, data: torch.Tensor, level: int) -> GpuCiphertext:
        """backend.py:86-92: divide-round by entry_primes[level] (NTT domain)."""
        return GpuCiphertext(self._rescale_data(data, level), level - 1)

    def _rescale_data(self, data: torch.Tensor, level: int) -> torch.Tensor:
        m = self._limbs(level)
        e = len(self.chain.entry_primes[level])
        polys = data.numel() // (m * self.n)
        out = self.chain.divround_ntt(data, polys, m, e)
        return out.view(*data.shape[:-2], m - e, self.n)

    def _to_ntt(self, coeff: torch.Tensor) -> torch.Tensor:
        return self.chain.ntt_fwd(coeff, coeff.shape[-2])

    def _to_coeff(self, data: torch.Tensor) -> torch.Tensor:
        return self.chain.ntt_inv(data.clone(), data.shape[-2])

    def _encode_rns(self, values, level: int, ntt: bool = False, scale: float = None,
                    limit: float = None) -> torch.Tensor:
        """encode (encoding.py:57-65) -> [limbs, N] residues at scale_at[level]
        (or an explicit scale); cached per value."""
        vals = np.asarray(values, dtype=np.float64)
        key = (vals.tobytes(), level, ntt, scale)
        hit = self._enc_cache.get(key)
        if hit is not None:
            self._enc_cache.move_to_end(key)
            return hit
        ch = self.chain
        m = self._limbs(level)
        sc = self._scale(level) if scale is None else scale
        lim = self._encode_limit if limit is None else limit
        if not self.encoder.host:  # one scatter + cuFFT + one finish kernel
            hb = _coeff_bound(vals, sc, self.n)
            fast = hb < lim and 4 * int(hb) < ch.modulus_at(level)
            res, mx = self.encoder.embed_residues(vals, sc, ch, m, need_max=not fast)
            res = res[0]
            if not fast:
                bound = float(mx.view(torch.float64).item())
                if bound >= lim:
                    raise self._errors.EncodingOverflow(
                        "scaled values exceed the exactly-representable coefficient range")
                if 4 * int(bound) >= ch.modulus_at(level):
                    raise self._errors.EncodingOverflow(
                        f"encoded coefficients (~2^{np.log2(bound + 1):.1f}) do not fit the "
                        f"current modulus with headroom")
            if ntt:
                ch.ntt_fwd(res, m)
            self._enc_cache[key] = res
            if len(self._enc_cache) > self._enc_cache_cap:
                self._enc_cache.popitem(last=False)
            return res
        coeffs = self.encoder.embed_device(vals, sc)
        # Every coefficient is (1/N) x a sum over the N spectrum entries (each
        # slot twice), so |c_j| <= scale * 2 sum|v| / N <= scale * max|v| (+ 1/2
        # from rounding): when that host-side bound already clears both checks,
        # skip the exact device max (a host sync per encode, not allowed inside
        # a graph capture); otherwise fall back to it — same error semantics.
        host_bound = _coeff_bound(vals, sc, self.n)
        if host_bound < lim and 4 * int(host_bound) < ch.modulus_at(level):
            res = ch.from_i64(coeffs.to(torch.int64), m)[0]
            if ntt:
                ch.ntt_fwd(res, m)
            self._enc_cache[key] = res
            if len(self._enc_cache) > self._enc_cache_cap:
                self._enc_cache.popitem(last=False)
            return res
        bound = float(coeffs.abs().max())
        if bound >= lim:
            raise self._errors.EncodingOverflow(
                "scaled values exceed the exactly-representable coefficient range")
        if 4 * int(bound) >= ch.modulus_at(level):
            raise self._errors.EncodingOverflow(
                f"encoded coefficients (~2^{np.log2(bound + 1):.1f}) do not fit the current "
                f"modulus with headroom")
        res = ch.from_i64(coeffs.to(torch.int64), m)[0]
        if ntt:
            ch.ntt_fwd(res, m)
        self._enc_cache[key] = res
        if len(self._enc_cache) > self._enc_cache_cap:
            self._enc_cache.popitem(last=False)
        return res

    def _check_encodable(self, values, level: int) -> None:
        """Deferred mode: raise EncodingOverflow at call time, as the eager
        encode would (encoding.py:46-48, 60-64).  The host-side bound clears
        almost every vector; the others are encoded exactly now."""
        vals = np.asarray(values, dtype=np.float64)
        hb = _coeff_bound(vals, self._scale(level), self.n)
        if hb < self._encode_limit and 4 * int(hb) < self.chain.modulus_at(level):
            return
        self._encode_rns(vals, level)

    def encode_many(self, items) -> None:
        """Batched _encode_rns for [(values, level, ntt)]: one FFT, one residue
        conversion and one NTT launch per (level, ntt) group, results stored in
        the encode cache the per-op calls read.  Vectors whose host-side bound
        does not clear the overflow checks are left to the exact per-op path."""
        groups: dict = {}
        for values, level, ntt in items:
            vals = np.asarray(values, dtype=np.float64)
            key = (vals.tobytes(), level, ntt, None)
            if key in self._enc_cache or vals.size == 0:
                continue
            grp = groups.setdefault((level, ntt), {})
            grp.setdefault(key, vals)
        ch = self.chain
        for (level, ntt), grp in groups.items():
            sc = self._scale(level)
            m = self._limbs(level)
            keys, rows = [], []
            for key, vals in grp.items():
                hb = _coeff_bound(vals, sc, self.n)
                if hb < self._encode_limit and 4 * int(hb) < ch.modulus_at(level):
                    keys.append(key)
                    rows.append(vals)
            if not keys:
                continue
            width = max(r.shape[0] for r in rows)
            mat = np.zeros((len(rows), width))
            for i, r in enumerate(rows):
                mat[i, : r.shape[0]] = r
            if self.encoder.host:
                res = ch.from_i64(self.encoder.embed_device_batch(mat, sc).to(torch.int64), m)
            else:
                res, _ = self.encoder.embed_residues(mat, sc, ch, m)  # [B, m, N]
            if ntt:
                ch.ntt_fwd(res, m)
            for i, key in enumerate(keys):
                self._enc_cache[key] = res[i]
            while len(self._enc_cache) > self._enc_cache_cap:
                self._enc_cache.popitem(last=False)

    # ------------------------------------------------------------------ hooks
    def _payload_elementwise(self, kind: str, a, b, out_level: int):
        if self._rec is not None:
            r = self._rec
            if kind.endswith("_ct"):
                ib = r.operand(b.payload)
            else:
                self._check_encodable(b.values if kind[:3] != "sub" else -b.values,
                                      a.level_remaining)
                ib = r.plaintext(b.values)
            return r.record(("ew", kind, None, r.operand(a.payload), ib), out_level)
        ch = self.chain
        ct_a: GpuCiphertext = a.payload
        op = kind[:3]
        if kind.endswith("_ct"):
            ct_b: GpuCiphertext = b.payload
            in_level = out_level + 1 if op == "mul" else out_level
            ct_a = self._adjust_to_level(ct_a, in_level)
            ct_b = self._adjust_to_level(ct_b, in_level)
            m = self._limbs(in_level)
            if op == "add":
                return GpuCiphertext(ch.add(ct_a.data, ct_b.data, m), in_level)
            if op == "sub":
                return GpuCiphertext(ch.sub(ct_a.data, ct_b.data, m), in_level)
            return self._mul_ct(ct_a, ct_b, in_level)
        in_level = ct_a.level
        m = self._limbs(in_level)
        if op == "mul":
            pt = self._encode_rns(b.values, in_level, ntt=True)
            x = ch.mul(ct_a.data, pt, m, b_rows=m)
            return self._rescale(x, in_level)
        pt = self._encode_rns(b.values if op == "add" else -b.values, in_level, ntt=True)
        out = ct_a.data.clone()
        ch.add(ct_a.data[0], pt, m, out=out[0])
        return GpuCiphertext(out, in_level)

    def _mul_ct(self, ct_a: GpuCiphertext, ct_b: GpuCiphertext, in_level: int) -> GpuCiphertext:
        """backend.py:136-143: tensor, relinearise, add, rescale — NTT domain."""
        out = self._hmult(ct_a.data.unsqueeze(0), ct_b.data.unsqueeze(0), in_level)
        return GpuCiphertext(out[0], in_level - 1)

    def _hmult(self, a: torch.Tensor, b: torch.Tensor, level: int) -> torch.Tensor:
        """[B, 2, m, N] x [B, 2, m, N] (NTT) -> [B, 2, m - e, N] (NTT)."""
        ch = self.chain
        m = self._limbs(level)
        bsz = a.shape[0]
        e = len(ch.entry_primes[level])
        d = ch.tensor(a, b, m)  # [B, 3, m, N]
        d2 = ch.ntt_from(d[:, 2], bsz, m, 3 * m * self.n, inverse=True)
        k = self._ks_k(level)
        key = self.relin_keys_k[k] if k != ch.k else self.relin_key
        if self._can_fold(m):  # d0 / d1 ride in the inner product as d*P
            acc = self._key_switch_acc(d2, m, batch=bsz, key=key, own=d[:, 2],
                                       own_stride=3 * m * self.n, k=k,
                                       fold=(d[:, 0], 3 * m * self.n, d[:, 1], 3 * m * self.n))
            out = ch.divround_ntt(acc, 2 * bsz, m + k, k, e, basis=ch.ext_basis(m, k))
            return out.view(bsz, 2, m - e, self.n)
        acc = self._key_switch_acc(d2, m, batch=bsz, key=key, own=d[:, 2],
                                   own_stride=3 * m * self.n, k=k)
        tail = d[:, 0:2, m - e:m].reshape(2 * bsz, e, self.n)
        out = ch.divround_ntt(acc, 2 * bsz, m + k, k, e, addend=d, addend_polys=2,
                              addend_period=2, addend_stride=3, addend_tail=tail,
                              basis=ch.ext_basis(m, k))
        return out.view(bsz, 2, m - e, self.n)

    def _payload_rotate(self, a, k: int):
        if self._rec is not None:
            r = self._rec
            return r.record(("rot", None, r.operand(a.payload), int(k)), a.level_remaining)
        ct: GpuCiphertext = a.payload
        if k == 0:
            return GpuCiphertext(ct.data.clone(), ct.level)
        galois = self.galois_for_step.get(k)
        if galois is None:
            galois = pow(5, k, 2 * self.n)
        key = self.rotation_key(galois)
        out = self._hrot(ct.data.unsqueeze(0), ct.level, galois=galois, key=key)
        return GpuCiphertext(out[0], ct.level)

    def _hrot(self, a: torch.Tensor, level: int, galois: int = 0, key: KeySwitchKey = None,
              g_items=None, key_ptrs=None, accumulate: bool = False) -> torch.Tensor:
        """backend.py:155-171 on [B, 2, m, N] NTT-domain ciphertexts: automorphism
        (a slot permutation in the NTT domain), key switch of c1', add c0'.
        accumulate: return a + rotate(a) instead — the add_ct of the
        rotate-and-sum schedules (packing.py:193-208) done in the ModDown
        combine pass, bit-identical to add_ct(a, rotate(a))."""
        ch = self.chain
        m = self._limbs(level)
        bsz = a.shape[0]
        r = ch.automorphism_ntt(a, galois, g_items=g_items, rows_per_item=2 * m)
        c1 = ch.ntt_from(r[:, 1], bsz, m, 2 * m * self.n, inverse=True)
        k = ch.k
        kk = self._ks_k(level)
        if key_ptrs is None and kk != ch.k and galois in self.rotation_keys_k[kk]:
            k, key = kk, self.rotation_keys_k[kk][galois]
        fold = (r[:, 0], 2 * m * self.n, None, 0) if self._can_fold(m) else None
        acc = self._key_switch_acc(c1, m, batch=bsz, key=key, key_ptrs=key_ptrs, own=r[:, 1],
                                   own_stride=2 * m * self.n, k=k, fold=fold)
        post = None
        if accumulate:
            post = a if a.is_contiguous() else a.contiguous()
        if fold is not None:  # c0' rode in the inner product as c0' * P
            out = ch.divround_ntt(acc, 2 * bsz, m + k, k, 0, basis=ch.ext_basis(m, k), post=post)
        else:
            out = ch.divround_ntt(acc, 2 * bsz, m + k, k, 0, addend=r, addend_polys=1,
                                  addend_period=2, addend_stride=2, basis=ch.ext_basis(m, k),
                                  post=post)
        return out.view(bsz, 2, m, self.n)

    def _encrypt_values(self, values, level: int, serial: int = None) -> GpuCiphertext:
        """backend.py:173-182: symmetric encryption, RNG (seed, serial); the
        result c0 = -a*s + NTT(m + e), c1 = a is the NTT form of the reference's."""
        return GpuCiphertext(self._encrypt_batch([values], level, [serial])[0], level)

    def _encrypt_batch(self, values_list, level: int, serials) -> torch.Tensor:
        """Encrypt several vectors at one level -> [B, 2, m, N]; serial None draws
        the next serial (the reference's default_rng((seed, serial)) stream)."""
        ch = self.chain
        primes = ch.limbs_at(level)
        m = len(primes)
        bsz = len(values_list)
        if bsz > 1:  # one batched encode for the whole batch (then cache hits)
            self.encode_many([(v, level, False) for v in values_list])
        msgs = []
        if self.sampler == "philox":
            srs = [next(self._serials) if sr is None else sr for sr in serials]
            seeds = _h2d(self.encryption_seeds(srs), self.device,
                         tag=("seeds", tuple(srs))).view(U64)
            a_d, e_d = ch.sample(seeds, m)
            msgs = [self._encode_rns(values, level) for values in values_list]
            out = torch.empty(bsz, 2, m, self.n, dtype=U64, device=self.device)
            out[:, 1].copy_(a_d)
            me = ch.from_i64(e_d, m)
            return self._finish_encrypt(out, me, msgs, m)
        a_np = np.empty((bsz, m, self.n), dtype=np.uint64)
        e_np = np.empty((bsz, self.n), dtype=np.int64)
        for i, (values, serial) in enumerate(zip(values_list, serials)):
            msgs.append(self._encode_rns(values, level))
            sr = next(self._serials) if serial is None else serial
            rng = np.random.default_rng((self.rng_seed, sr))
            for j, p in enumerate(primes):
                a_np[i, j] = rng.integers(0, p, self.n, dtype=np.uint64)
            e_np[i] = np.rint(rng.normal(0.0, ERROR_SIGMA, self.n)).astype(np.int64)
        out = torch.empty(bsz, 2, m, self.n, dtype=U64, device=self.device)
        out[:, 1].copy_(torch.from_numpy(a_np))
        me = ch.from_i64(_h2d(e_np, self.device), m)  # [B, m, N]
        return self._finish_encrypt(out, me, msgs, m)

    def encryption_seeds(self, serials) -> np.ndarray:
        """Philox keys of the encryptions with these serials (one stream per
        (rng_seed, serial), the device analogue of default_rng((seed, serial)))."""
        return np.array([_mix64(self.rng_seed, 0x454E43, sr) for sr in serials], dtype=np.int64)

    def _finish_encrypt(self, out, me, msgs, m):
        """c1 = a (NTT domain), c0 = NTT(m + e) - a*s."""
        ch = self.chain
        ch.add(me, torch.stack(msgs), m, out=me)
        ch.ntt_fwd(me, m)
        a_s = ch.mul(out[:, 1].contiguous(), self.sk.s_full[:m], m, b_rows=m)
        out[:, 0].copy_(ch.sub(me, a_s, m))
        return out

    def _payload_encrypt(self, pv, level: int, serial: int):
        if self._rec is not None:  # the RNG serial the eager call would draw
            self._check_encodable(pv.values, level)
            r = self._rec
            return r.record(("enc", None, r.plaintext(pv.values)), level,
                            serial=next(self._serials))
        return self._encrypt_values(pv.values, level)

    def _phase(self, ct: GpuCiphertext) -> torch.Tensor:
        """c0 + c1*s, coefficient domain."""
        ch = self.chain
        m = ct.data.shape[1]
        t = ch.mul(ct.data[1], self.sk.s_full[:m], m)
        ch.add(ct.data[0], t, m, out=t)
        return ch.ntt_inv(t, m)

    def _decrypt_values(self, ct: GpuCiphertext) -> np.ndarray:
        """backend.py:187-190: phase, centered CRT lift, decode."""
        m = ct.data.shape[1]
        coeffs = self.chain.to_f64(self._phase(ct), m)[0]
        return self.encoder.unembed_device(coeffs, self._scale(ct.level)).cpu().numpy()

    def _decrypt_values_batch(self, data: torch.Tensor, level: int) -> np.ndarray:
        """[B, 2, m, N] ciphertexts at one level -> [B, N/2] slot values: the
        reference's per-item decrypt (backend.py:187-190) with one phase
        computation, one CRT lift, one FFT and one device->host copy."""
        ch = self.chain
        b, _, m, n = data.shape
        c1 = data[:, 1].contiguous()
        t = ch.mul(c1, self.sk.s_full[:m], m, b_rows=m)
        ch.add(data[:, 0].contiguous(), t, m, out=t)
        ch.ntt_inv(t, m)
        coeffs = ch.to_f64(t, m)  # [B, N]
        return self.encoder.unembed_device(coeffs, self._scale(level)).cpu().numpy()

    def decrypt_complex(self, ct: GpuCiphertext, scale: float = None) -> np.ndarray:
        """Complex slot values (the reference decodes real parts only)."""
        m = ct.data.shape[1]
        coeffs = self.chain.to_f64(self._phase(ct), m)[0]
        w = coeffs.to(torch.complex128) * self.encoder.twist
        spec = torch.fft.ifft(w) * self.n
        sc = self._scale(ct.level) if scale is None else scale
        return (spec[self.encoder.bins] / sc).cpu().numpy()

    def _payload_decrypt(self, cv):
        if self._rec is not None:
            return self._decrypt_values(self._rec.resolve(cv.payload))
        return self._decrypt_values(cv.payload)

    def _payload_bootstrap(self, cv, serial: int):
        """Custodian refresh (backend.py:195-206): decrypt, optional U(+-eps),
        re-encrypt at refresh_level.  With real_bootstrap=True the ciphertext is
        instead dropped to level 0 and bootstrapped homomorphically
        (bootstrap.py); the serial is still consumed as the refresh would."""
        if self._rec is not None:  # one serial, as either eager form draws
            r = self._rec
            return r.record(("bs", None, r.operand(cv.payload)), self.params.refresh_level,
                            serial=next(self._serials))
        if self.real_bootstrap:
            next(self._serials)
            return self.bootstrap_ct(cv.payload)
        values = self._decrypt_values(cv.payload)
        if self.bootstrap_eps > 0.0:
            values = values + self._bs_rng.uniform(-self.bootstrap_eps, self.bootstrap_eps,
                                                   values.shape[0])
        return self._encrypt_values(values, self.params.refresh_level)

    # ------------------------------------------------------------ serialization
    def serialize_cipher(self, cv) -> bytes:
        """RBCT (backend.py:210-222): header then c0, c1 coefficient planes, LE u64."""
        ct: GpuCiphertext = cv.payload
        if self._rec is not None:
            ct = self._rec.resolve(ct)
        head = struct.pack("<4sIQId", CT_MAGIC, SERIAL_VERSION, self.n, ct.level, cv.scale_bits)
        body = self._to_coeff(ct.data).cpu().numpy().astype("<u8").tobytes()
        return head + body

    def deserialize_cipher(self, blob: bytes):
        fmt = "<4sIQId"
        hs = struct.calcsize(fmt)
        E = self._errors
        if len(blob) < hs:
            raise E.SerializationError("truncated ciphertext header")
        magic, version, degree, level, scale_bits = struct.unpack(fmt, blob[:hs])
        if magic != CT_MAGIC:
            raise E.SerializationError(f"bad ciphertext magic {magic!r}")
        if version != SERIAL_VERSION:
            raise E.SerializationError(f"unsupported ciphertext version {version}")
        if degree != self.n:
            raise E.SerializationError("ciphertext degree does not match parameters")
        if not 0 <= level <= self.params.level:
            raise E.SerializationError(f"ciphertext level {level} out of range")
        m = self._limbs(level)
        body = blob[hs:]
        if len(body) != 2 * m * degree * 8:
            raise E.SerializationError("ciphertext body length mismatch")
        arr = np.frombuffer(body, dtype="<u8").reshape(2, m, degree).astype(np.uint64)
        data = self._to_ntt(torch.from_numpy(arr).to(self.device))
        rl = self.params.refresh_level
        return self._api.CipherVector(
            payload=GpuCiphertext(data, level), level_remaining=level, scale_bits=scale_bits,
            depth=rl - level if level < rl else 0, backend_id=self.backend_id,
            keyset_id=self.keyset_id, serial=next(self._serials))

    # ------------------------------------------------------ bootstrapping helpers
    def encode_complex_ntt(self, z, level: int, scale: float = None) -> torch.Tensor:  # noqa: D401
        """Complex slot vector -> NTT-domain plaintext [limbs(level), N] at
        scale_at[level] (or `scale`)."""
        ch = self.chain
        m = self._limbs(level)
        coeffs = self.encoder.embed_complex_device(z, self._scale(level) if scale is None
                                                   else scale)
        # bootstrapping plaintexts are encoded at ~q_level (up to 2^61): float64
        # rounding then costs 2^-52 relative, far below the ciphertext noise
        if float(coeffs.abs().max()) >= float(2**62):
            raise self._errors.EncodingOverflow("complex plaintext exceeds 2^62")
        res = ch.from_i64(coeffs.to(torch.int64), m)[0]
        return ch.ntt_fwd(res, m)

    def monomial_ntt(self, power: int, level: int) -> torch.Tensor:
        """NTT form of X^power over the limbs of `level` (cached)."""
        key = ("mono", power, level)
        hit = self._adjust_cache.get(key)
        if hit is None:
            ch = self.chain
            m = self._limbs(level)
            c = torch.zeros(self.n, dtype=torch.int64, device=self.device)
            c[power % self.n] = -1 if (power // self.n) % 2 else 1
            hit = ch.publish(ch.ntt_fwd(ch.from_i64(c, m)[0], m))
            self._adjust_cache[key] = hit
        return hit

    def hoisted_rotations(self, data: torch.Tensor, level: int, galois_list,
                          stack: bool = False, streams=None):
        """Rotate ciphertexts ([..., 2, m, N], NTT domain) by several Galois
        elements sharing a single ModUp: the digits are lifted and transformed
        once and permuted per rotation in the NTT domain (an automorphism
        commutes with the basis extension up to multiples of Q_j, which the key
        switch absorbs as noise).  stack=True returns one tensor
        [len(galois_list), ..., 2, m, N] instead of a list.  streams: side
        streams the rotations are spread over (independent after the ModUp)."""
        ch = self.chain
        m = self._limbs(level)
        ext = m + ch.k
        lead = data.shape[:-3]
        d = data.reshape(-1, 2, m, self.n)
        b = d.shape[0]
        c1 = ch.ntt_from(d[:, 1], b, m, 2 * m * self.n, inverse=True)
        digits = ch.modup(c1, m, self.alpha, self._bconv(m), batch=b)
        ch.ntt_fwd(digits, ext, ch.ext_map(m))
        c0s = d[:, 0].contiguous()
        res = torch.empty(len(galois_list), b, 2, m, self.n, dtype=U64, device=self.device)
        main = torch.cuda.current_stream()
        for st in streams or ():
            st.wait_stream(main)
        for i, g in enumerate(galois_list):
            key = self.rotation_key(g)
            ctx = torch.cuda.stream(streams[i % len(streams)]) if streams else _nullctx()
            with ctx:
                dg = ch.automorphism_ntt(digits, g)
                acc = ch.ks_inner(dg, m, self.alpha, key=key.data)
                c0 = ch.automorphism_ntt(c0s, g)
                ch.divround_ntt(acc, 2 * b, ext, ch.k, 0, addend=c0, addend_polys=1,
                                addend_period=2, addend_stride=1, basis=ch.ext_basis(m),
                                out=res[i].view(2 * b, m, self.n))
        for st in streams or ():
            main.wait_stream(st)
        res = res.view(len(galois_list), *lead, 2, m, self.n)
        return res if stack else list(res.unbind(0))

    def prepare_bootstrap(self) -> None:
        """Build the bootstrapper's device tables (plaintext diagonals, basis
        constants, FFT plans) ahead of the first refresh — setup work, like key
        generation — by bootstrapping an encryption of zeros once."""
        if not self.real_bootstrap:
            return
        ct = GpuCiphertext(self._encrypt_batch([np.zeros(self.n // 2)], 0, [None])[0], 0)
        self.bootstrap_ct(ct)

    def bootstrap_batch(self, data: torch.Tensor, level: int) -> torch.Tensor:
        """Bootstrap a batch [B, 2, m, N] of ciphertexts at one level together:
        every stage runs once over the batch (the refreshed weights of a
        training step are independent).  Returns [B, 2, m(refresh), N]."""
        return self.bootstrap_ct(GpuCiphertext(data, level)).data

    def bootstrap_ct(self, ct: GpuCiphertext) -> GpuCiphertext:
        """Homomorphic bootstrapping of a payload (any level) to refresh_level
        (always over the full special modulus)."""
        prev, self._force_full_p = self._force_full_p, True
        try:
            return self._bootstrap_ct(ct)
        finally:
            self._force_full_p = prev

    def _bootstrap_ct(self, ct: GpuCiphertext) -> GpuCiphertext:
        if self._bootstrapper is None:
            from .bootstrap import Bootstrapper

            self._bootstrapper = Bootstrapper(self)
        if ct.level > 0:
            ct = GpuCiphertext(self._adjust_data(ct.data, ct.level, 0), 0)
        return self._bootstrapper.bootstrap(ct)

    def rotate_data(self, data: torch.Tensor, level: int, galois: int) -> torch.Tensor:
        """[..., 2, m, N] -> the same, every item rotated by one Galois element."""
        m = self._limbs(level)
        out = self._hrot(data.reshape(-1, 2, m, self.n), level, galois=galois,
                         key=self.rotation_key(galois))
        return out.view(*data.shape[:-3], 2, m, self.n)

    def mod_raise(self, ct: GpuCiphertext) -> GpuCiphertext:
        """Bootstrapping step 1: reinterpret a level-0 ciphertext (one limb q0)
        modulo the full chain Q_L by centred lifting of its coefficients."""
        ch = self.chain
        m0 = self._limbs(ct.level)
        if ct.level != 0 or m0 != 1:
            raise self._errors.IncompatibleOperands("mod_raise needs a one-limb level-0 ciphertext")
        top = self.params.level
        m = self._limbs(top)
        lead = ct.data.shape[:-3]
        coeff = ch.ntt_inv(ct.data.clone(), 1)
        polys = coeff.numel() // self.n
        out = torch.empty(polys, 1, m, self.n, dtype=U64, device=self.device)
        from . import _native as nat

        basis = tuple(range(m))
        nat.check(nat.LIB.ckb_modup(ch.ring_p, nat.ptr(out), nat.ptr(coeff), 0, polys, 1,
                                    ch.q_map(1), m, ch.cmap(basis), 1, None, 0,
                                    nat.stream_handle()), "mod_raise")
        data = out.view(*lead, 2, m, self.n)
        return GpuCiphertext(ch.ntt_fwd(data, m), top)

    # ------------------------------------------------------------ batched engine
    # One launch per stage across a whole batch of ciphertexts (the
    # config-2 workload: 64 independent ciphertexts).  Same
    # arithmetic as the per-ciphertext hooks, which are these with B = 1.

    def batch_hmult(self, a: torch.Tensor, b: torch.Tensor, level: int) -> torch.Tensor:
        """ct x ct multiply + relinearise + rescale of B pairs at one level.
        a, b: [B, 2, limbs(level), N] NTT domain -> [B, 2, limbs(level-1), N]."""
        return self._hmult(a, b, level)

    def _rotation_tables(self, steps):
        key = tuple(int(s) for s in steps)
        cache = self.__dict__.setdefault("_rot_tab_cache", {})
        if key not in cache:
            slots = self.params.slot_count
            two_n = 2 * self.n
            gal = [self.galois_for_step.get(s % slots, pow(5, s % slots, two_n)) for s in key]
            keys = [self.rotation_key(g) for g in gal]
            g_items = self.chain.upload_table(np.array(gal, dtype=np.int64)).view(U64)
            ptrs = self.chain.upload_table(np.array([k.data.data_ptr() for k in keys],
                                                    dtype=np.int64))
            cache[key] = (g_items, ptrs, keys)
        return cache[key]

    def batch_hrot(self, a: torch.Tensor, steps, level: int) -> torch.Tensor:
        """Rotate item i of a [B, 2, limbs, N] NTT-domain batch left by steps[i]."""
        g_items, ptrs, _ = self._rotation_tables(steps)
        return self._hrot(a, level, g_items=g_items, key_ptrs=ptrs)

    def pack_batch(self, data: torch.Tensor, level: int) -> torch.Tensor:
        """[B, 2, limbs(level), N] payload batch -> [B, bytes] uint8 in the packed
        transfer format (ckb_pack: 5 bytes per residue of a prime < 2^40), for
        host <-> device copies of ciphertext batches (streaming.Pipeline)."""
        m = self._limbs(level)
        b = data.shape[0]
        return self.chain.pack(data.contiguous(), 2 * b, m).view(b, -1)

    def unpack_batch(self, packed: torch.Tensor, level: int) -> torch.Tensor:
        """Inverse of pack_batch: [B, bytes] uint8 -> [B, 2, limbs(level), N]."""
        m = self._limbs(level)
        b = packed.shape[0]
        return self.chain.unpack(packed.contiguous(), 2 * b, m).view(b, 2, m, self.n)

    def batch_ntt(self, a: torch.Tensor, level: int, inverse: bool = False) -> torch.Tensor:
        """In-place NTT / iNTT of every limb of a [..., limbs(level), N] batch."""
        m = self._limbs(level)
        return self.chain.ntt_inv(a, m) if inverse else self.chain.ntt_fwd(a, m)

    # ---------------------------------------------------------------- raw access
    def payload_from_planes(self, planes: np.ndarray, level: int) -> GpuCiphertext:
        """Wrap host (2, limbs, N) coefficient-domain planes (RBCT order) as a payload."""
        t = torch.from_numpy(np.ascontiguousarray(planes, dtype=np.uint64)).to(self.device)
        return GpuCiphertext(self._to_ntt(t), level)

    def planes_of(self, payload: GpuCiphertext) -> np.ndarray:
        """Coefficient-domain (2, limbs, N) planes of a payload (RBCT order)."""
        if self._rec is not None:
            payload = self._rec.resolve(payload)
        return self._to_coeff(payload.data).cpu().numpy()


_nullctx = contextlib.nullcontext


def _coeff_bound(vals: np.ndarray, scale: float, n: int) -> float:
    """Upper bound on |coefficient| of the encoding of real slots vals at scale
    (encoding.py:34-49: coefficients are spectrum sums / N, each slot twice)."""
    if not vals.size:
        return 0.0
    a = np.abs(vals)
    return scale * min(float(np.max(a)), 2.0 * float(np.sum(a)) / n) * (1 + 1e-9) + 1.0


def _mix64(*parts) -> int:
    """splitmix64-style hash of integers -> a 64-bit Philox key (signed for torch)."""
    x = 0x9E3779B97F4A7C15
    for v in parts:
        x = (x ^ (int(v) & 0xFFFFFFFFFFFFFFFF)) * 0xBF58476D1CE4E5B9 & 0xFFFFFFFFFFFFFFFF
        x = (x ^ (x >> 31)) * 0x94D049BB133111EB & 0xFFFFFFFFFFFFFFFF
        x ^= x >> 29
    return x - (1 << 64) if x >= 1 << 63 else x


def _hw_secret(n: int, h: int, seed: int) -> np.ndarray:
    """Ternary secret with exactly h non-zeros (+-1), positions and signs from
    default_rng((seed, 0x5EC7)) — BASELINE configs' HW-64 / HW-192 secrets."""
    if not 0 < h <= n:
        raise he_errors.InvalidParameters(f"secret Hamming weight {h} out of range")
    rng = np.random.default_rng((seed, 0x5EC7))
    s = np.zeros(n, dtype=np.int64)
    pos = rng.choice(n, size=h, replace=False)
    s[pos] = rng.choice(np.array([-1, 1], dtype=np.int64), size=h)
    return s


class B200Backend(B200CkksCore, he_api.Backend):
    """The B200 CKKS backend bound to this package's HE API mirror."""


def save_custodian(custodian) -> bytes:
    """RBKY key container (backend.py:250-271): params, rotations, seed, eps, secret."""
    be = custodian.backend
    if not isinstance(be, B200CkksCore):
        raise he_errors.SerializationError("key files apply to the CKKS backend")
    out = io.BytesIO()
    out.write(struct.pack("<4sIQ", KEY_MAGIC, SERIAL_VERSION, be.params.poly_degree))
    out.write(be.params.digest())
    blob = json.dumps(dataclasses.asdict(be.params), sort_keys=True).encode()
    out.write(struct.pack("<I", len(blob)))
    out.write(blob)
    rots = sorted(be.rotation_indices)
    out.write(struct.pack("<I", len(rots)))
    out.write(struct.pack(f"<{len(rots)}q", *rots))
    out.write(struct.pack("<qd", be.rng_seed, be.bootstrap_eps))
    out.write(be.sk.coeffs.astype("<i1").tobytes())
    return out.getvalue()


def load_custodian(blob: bytes, **backend_options):
    """Inverse of save_custodian; evaluation keys are regenerated (backend.py:274-293)."""
    from .scheme import SchemeParams

    buf = io.BytesIO(blob)
    magic, version, degree = struct.unpack("<4sIQ", buf.read(16))
    if magic != KEY_MAGIC:
        raise he_errors.SerializationError(f"bad key magic {magic!r}")
    if version != SERIAL_VERSION:
        raise he_errors.SerializationError(f"unsupported key version {version}")
    digest = buf.read(32)
    (n_params,) = struct.unpack("<I", buf.read(4))
    raw = json.loads(buf.read(n_params).decode())
    raw["modulus_chain"] = tuple(raw["modulus_chain"])
    params = SchemeParams(**raw)
    if params.digest() != digest:
        raise he_errors.SerializationError("key file parameter digest mismatch")
    (n_rots,) = struct.unpack("<I", buf.read(4))
    rots = struct.unpack(f"<{n_rots}q", buf.read(8 * n_rots))
    seed, eps = struct.unpack("<qd", buf.read(16))
    secret = np.frombuffer(buf.read(degree), dtype="<i1").astype(np.int64)
    be = B200Backend(params, rotation_indices=rots, rng_seed=seed, bootstrap_eps=eps,
                     _secret=secret, **backend_options)
    return he_api.KeyCustodian(be, rots)
