"""pytest plugin: run the reference's OWN tests with the B200 backend swapped in.

Loaded with ``-p ref_plugin`` by tests/test_gpu_reference_suite.py on a
subprocess pytest over baseline/_ref/ref_tests (the unmodified reference test
modules, vendored by tools/vendor_reference.py).  At configure time, before
any reference test module is imported, ``plugin.install()`` replaces
``ciphermlp.ckks.backend.CkksBackend`` (resolved at call time by
``keygen(..., backend="ckks")`` and ``load_custodian``, api.py:343-346,
ckks/backend.py:291), so every CKKS object those tests build is the B200
backend.  Options for the installed class come from CKB_REF_PLUGIN_OPTS
(JSON; default: the reference's own prime layout and samplers).

At session end the plugin writes how many B200 backends the tests built and
the class that was installed to CKB_REF_PLUGIN_REPORT, so the caller can
prove the run did not silently use the reference's numpy backend.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_STATE = {"built": 0, "cls": None}


def pytest_configure(config):
    import ciphermlp.ckks.backend as rb

    config.addinivalue_line("markers", "slow: the reference's long-running tests")
    from paper_2506_19693_b200 import plugin

    opts = json.loads(os.environ.get("CKB_REF_PLUGIN_OPTS", "{}"))
    cls, _old = plugin.install(**opts)
    base_init = cls.__init__

    def __init__(self, *a, **kw):
        base_init(self, *a, **kw)
        _STATE["built"] += 1

    cls.__init__ = __init__
    _STATE["cls"] = f"{cls.__module__}.{cls.__qualname__}"
    assert rb.CkksBackend is cls


def pytest_report_header(config):
    return f"ciphermlp.ckks.backend.CkksBackend -> {_STATE['cls']} (B200 sm_100a kernels)"


def pytest_sessionfinish(session, exitstatus):
    import ciphermlp.ckks.backend as rb

    path = os.environ.get("CKB_REF_PLUGIN_REPORT")
    if path:
        from paper_2506_19693_b200 import _native

        with open(path, "w") as fh:
            json.dump({"b200_backends_built": _STATE["built"], "installed": _STATE["cls"],
                       "still_installed": rb.CkksBackend.__module__ ==
                       "paper_2506_19693_b200.plugin",
                       "native_library": _native._LIB_PATH,
                       "exitstatus": int(exitstatus)}, fh)
