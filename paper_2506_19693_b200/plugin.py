"""Drop-in registration into the reference package.

The reference resolves its CKKS backend class at call time
(/root/reference/pkg/src/ciphermlp/api.py:343-346, ckks/backend.py:291), so
replacing ``ciphermlp.ckks.backend.CkksBackend`` reroutes ``keygen(...,
backend="ckks")``, ``load_custodian``, ``training.build_run`` and the whole
layer stack (packing, linalg, nn, training) onto the B200 kernels with no
edits to the reference.  The installed class is the same payload core as
``backend.B200Backend`` bound to the reference's own ``Backend`` base, raising
the reference's exception types and building its ``CipherVector``.
"""

from __future__ import annotations


def make_backend_class(ciphermlp_pkg=None):
    import importlib

    from .backend import B200CkksCore

    cm = ciphermlp_pkg or importlib.import_module("ciphermlp")
    api = importlib.import_module(cm.__name__ + ".api")
    errors = importlib.import_module(cm.__name__ + ".errors")
    return type("CkksBackend", (B200CkksCore, api.Backend),
                {"_errors": errors, "_api": api, "__module__": __name__,
                 "__doc__": "B200 RNS-CKKS backend installed into ciphermlp."})


def install(ciphermlp_pkg=None, **default_options):
    """Replace ciphermlp.ckks.backend.CkksBackend; returns (new_class, old_class).

    ``default_options`` (e.g. prime_layout="baseline", dnum=3) are applied to
    every backend the reference constructs."""
    import functools
    import importlib

    cls = make_backend_class(ciphermlp_pkg)
    if default_options:
        base_init = cls.__init__

        @functools.wraps(base_init)
        def __init__(self, *a, **kw):
            for k, v in default_options.items():
                kw.setdefault(k, v)
            base_init(self, *a, **kw)

        cls.__init__ = __init__
    mod = importlib.import_module((ciphermlp_pkg.__name__ if ciphermlp_pkg else "ciphermlp")
                                  + ".ckks.backend")
    old = mod.CkksBackend
    mod.CkksBackend = cls
    return cls, old


def uninstall(old_class, ciphermlp_pkg=None):
    import importlib

    mod = importlib.import_module((ciphermlp_pkg.__name__ if ciphermlp_pkg else "ciphermlp")
                                  + ".ckks.backend")
    mod.CkksBackend = old_class
