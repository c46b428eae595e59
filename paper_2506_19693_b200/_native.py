"""ctypes binding of the sm_100a kernel library (include/ckks_b200.h).

This is the FFI a maintainer of the reference would add.
There is deliberately no fallback: if the library is missing or fails to load,
importing the backend raises, and every op raises if a kernel launch fails.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_LIB_PATH = os.environ.get("CKB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "_lib", "libckks_b200.so")

c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_vp = ctypes.c_void_p


class CkbRing(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n_primes", ctypes.c_uint32),
                ("mods", c_vp), ("ntt", c_vp), ("pair", c_vp),
                ("f64_mask", ctypes.c_uint64 * 2), ("ntt_chunk_bytes", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("wide_mask", ctypes.c_uint64 * 2), ("mid_mask", ctypes.c_uint64 * 2)]


RING_HPS_EXACT = 1  # ckb_ring.flags (include/ckks_b200.h)
RING_NTT_SPLIT = 2
RING_TC = 4  # tensor-core ModUp / ModDown correction (needs wide_mask)
RING_LAZY_BCONV = 8  # their outputs in [0, 3p): forward-NTT inputs only
DEFAULT_NTT_CHUNK_BYTES = 96 << 20


F64_PRIME_LIMIT = 1 << 46  # csrc/ntt.cu: primes below run the FP64 butterflies


def f64_mask(primes) -> tuple:
    m = 0
    for i, p in enumerate(primes):
        if int(p) < F64_PRIME_LIMIT and i < 128:
            m |= 1 << i
    return (m & (2**64 - 1), m >> 64)


TC_MID_LIMIT = 1 << 40   # csrc/tc.cu column classes: < 2^40: 5 byte columns,
TC_WIDE_LIMIT = 1 << 48  # [2^40, 2^48): 6, >= 2^48: 8


def _mask(primes, lo, hi) -> tuple:
    m = 0
    for i, p in enumerate(primes):
        if lo <= int(p) < hi and i < 128:
            m |= 1 << i
    return (m & (2**64 - 1), m >> 64)


def wide_mask(primes) -> tuple:
    return _mask(primes, TC_WIDE_LIMIT, 1 << 64)


def mid_mask(primes) -> tuple:
    return _mask(primes, TC_MID_LIMIT, TC_WIDE_LIMIT)


class NativeError(RuntimeError):
    pass


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"B200 kernel library not built: {_LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback.")
    lib = ctypes.CDLL(_LIB_PATH)
    R = ctypes.POINTER(CkbRing)
    sig = {
        "ckb_version": ([], ctypes.c_int),
        "ckb_build_tables": ([ctypes.c_uint32, c_u64p, ctypes.c_uint32, c_u64p, c_u64p, c_u64p],
                             ctypes.c_int),
        "ckb_ntt_forward": ([R, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_ntt_inverse": ([R, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_ntt_forward_combine": ([R, c_vp, c_vp, c_vp, ctypes.c_int64, c_vp, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     c_i32p, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp,
                                     ctypes.c_int64, c_vp], ctypes.c_int),
        "ckb_ntt_forward_from": ([R, c_vp, c_vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                  c_i32p, c_vp], ctypes.c_int),
        "ckb_ntt_inverse_from": ([R, c_vp, c_vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                  c_i32p, c_vp], ctypes.c_int),
        "ckb_elementwise": ([R, ctypes.c_int, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int,
                             c_i32p, ctypes.c_int, c_vp], ctypes.c_int),
        "ckb_scalar_mac": ([R, c_vp, ctypes.POINTER(c_vp), c_i32p, c_vp, ctypes.c_int,
                            ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_pt_mac": ([R, c_vp, c_vp, c_vp, ctypes.c_int64, c_i32p, c_vp, ctypes.c_int64,
                        ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_scalar_mul": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_u64p, c_vp],
                           ctypes.c_int),
        "ckb_tensor": ([R, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp],
                       ctypes.c_int),
        "ckb_ks_ntt_mac": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            c_i32p, c_i32p, c_vp, ctypes.c_int64, c_vp, c_vp, ctypes.c_int,
                            c_i32p, c_vp], ctypes.c_int),
        "ckb_embed_scatter": ([c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                               ctypes.c_double, c_vp, ctypes.c_int, c_vp], ctypes.c_int),
        "ckb_embed_finish": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp, c_vp,
                              c_vp], ctypes.c_int),
        "ckb_modup": ([R, c_vp, c_vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, c_i32p,
                       ctypes.c_int, c_i32p, ctypes.c_int, c_vp, ctypes.c_int, c_vp],
                      ctypes.c_int),
        "ckb_ks_inner": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i32p,
                          ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int64, c_vp, c_vp,
                          ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_ks_inner_fold": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i32p,
                               ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int64, c_vp, c_vp,
                               ctypes.c_int, c_i32p, c_vp, ctypes.c_int64, c_vp, ctypes.c_int64,
                               c_vp, ctypes.c_int, c_vp], ctypes.c_int),
        "ckb_divround": ([R, c_vp, c_vp, ctypes.c_int64, c_vp, ctypes.c_int, ctypes.c_int,
                          ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i32p, ctypes.c_int,
                          ctypes.c_int, c_u64p, c_vp, c_vp, c_vp],
                         ctypes.c_int),
        "ckb_automorphism": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, ctypes.c_uint64,
                              c_vp, ctypes.c_int, c_vp], ctypes.c_int),
        "ckb_from_i64": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_to_f64": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_divround_ntt_corr": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i32p,
                                   ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp],
                                  ctypes.c_int),
        "ckb_divround_ntt_combine": ([R, c_vp, c_vp, ctypes.c_int64, c_vp, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int,
                                      ctypes.c_int, c_i32p, ctypes.c_int, ctypes.c_int, c_vp,
                                      c_vp, c_vp], ctypes.c_int),
        "ckb_divround_ntt_combine_acc": ([R, c_vp, c_vp, ctypes.c_int64, c_vp, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int,
                                          ctypes.c_int, c_i32p, ctypes.c_int, ctypes.c_int, c_vp,
                                          c_vp, c_vp, ctypes.c_int64, c_vp], ctypes.c_int),
        "ckb_automorphism_ntt": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_uint64, c_vp,
                                  ctypes.c_int, c_vp], ctypes.c_int),
        "ckb_reduce": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_sample": ([R, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, ctypes.c_double,
                        c_vp], ctypes.c_int),
        "ckb_packed_bytes": ([R, ctypes.c_int, ctypes.c_int, c_i32p], ctypes.c_int64),
        "ckb_pack": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_unpack": ([R, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_i32p, c_vp], ctypes.c_int),
        "ckb_tc_probe": ([ctypes.c_int, ctypes.c_int, c_vp, c_vp], ctypes.c_int),
        "ckb_tc_selftest": ([c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_vp], ctypes.c_int),
        "ckb_alu_probe": ([ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, c_vp,
                           c_vp], ctypes.c_int),
        "ckb_alu_probe_f64": ([ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                               c_vp, c_vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("CKB_LIB") and not hasattr(lib, name):
            continue  # A/B runs against an older build (tools/): missing entry points unused
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.ckb_version() != 1:
        raise ImportError("libckks_b200.so version mismatch; rebuild")
    return lib


LIB = _load()
EXPORTED = ("ckb_version", "ckb_build_tables", "ckb_ntt_forward", "ckb_ntt_inverse",
            "ckb_ntt_forward_combine", "ckb_ntt_forward_from", "ckb_ntt_inverse_from",
            "ckb_elementwise", "ckb_pt_mac", "ckb_scalar_mac", "ckb_scalar_mul", "ckb_tensor", "ckb_modup", "ckb_ks_inner", "ckb_ks_inner_fold", "ckb_ks_ntt_mac", "ckb_embed_scatter", "ckb_embed_finish",
            "ckb_divround", "ckb_automorphism", "ckb_from_i64", "ckb_to_f64",
            "ckb_divround_ntt_corr", "ckb_divround_ntt_combine", "ckb_divround_ntt_combine_acc",
            "ckb_automorphism_ntt",
            "ckb_reduce", "ckb_sample", "ckb_alu_probe",
            "ckb_alu_probe_f64", "ckb_tc_selftest", "ckb_tc_probe", "ckb_packed_bytes", "ckb_pack",
            "ckb_unpack")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what} failed with status {rc}")


def build_tables(log_n: int, primes) -> tuple:
    """Host tables for ckb_ring (see include/ckks_b200.h)."""
    n = 1 << log_n
    np_ = len(primes)
    pr = np.ascontiguousarray(np.array(primes, dtype=np.uint64))
    mods = np.zeros((np_, 16), dtype=np.uint64)
    ntt = np.zeros((np_, 4, n), dtype=np.uint64)
    pair = np.zeros((np_, np_, 4), dtype=np.uint64)
    rc = LIB.ckb_build_tables(log_n, pr.ctypes.data_as(c_u64p), np_, mods.ctypes.data_as(c_u64p),
                              ntt.ctypes.data_as(c_u64p), pair.ctypes.data_as(c_u64p))
    check(rc, "ckb_build_tables")
    return mods, ntt, pair


def i32_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_int32 * len(vals))(*vals)


def u64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_uint64 * len(vals))(*vals)


def ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle():
    """The caller's current CUDA stream (every launch goes on it).  The raw
    accessor avoids constructing a torch.cuda.Stream object per launch, which
    dominated the host cost of small-ring (N=2^12) programs."""
    if _raw_stream is not None:
        return ctypes.c_void_p(_raw_stream(torch._C._cuda_getDevice()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
