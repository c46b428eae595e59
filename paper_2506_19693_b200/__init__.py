"""B200-native RNS-CKKS backend for ReBoot encrypted training (arxiv 2506.19693).

Public surface mirrors the reference package ``ciphermlp``'s HE API
(he_api.py, scheme.py, he_errors.py); the backend itself (backend.py) runs every
ciphertext operation in hand-written sm_100a kernels (csrc/, include/ckks_b200.h).

    from paper_2506_19693_b200 import keygen, make_params, make_plain
    cust = keygen(make_params(level=8, scale_bits=40, poly_degree=4096), {1, -1},
                  prime_layout="baseline", secret_hw=64)

``plugin.install()`` swaps the backend into an installed reference package
(``ciphermlp.ckks.backend.CkksBackend``) so its layer code runs unchanged.
"""

from .he_api import (CipherVector, DepthLedger, Evaluator, KeyCustodian, PlainVector, keygen,
                     make_plain)
from .scheme import INSECURE, SchemeParams, make_params

__all__ = ["CipherVector", "DepthLedger", "Evaluator", "KeyCustodian", "PlainVector", "keygen",
           "make_plain", "INSECURE", "SchemeParams", "make_params"]


def backend_class():
    from .backend import B200Backend

    return B200Backend
