"""RBOT model container (model_io, mirroring ciphermlp/serialize.py:38-107)
against the reference's own container in tests/golden/ref_rbot_n512.npz.

CPU part: the container layer alone, with a pass-through backend whose
ciphertexts are the raw RBCT blobs — parse, re-emit byte for byte, and the
reference's error cases.  GPU part: the same blob through the B200 backend
(RBKY key file -> custodian, RBCT payloads -> device ciphertexts): decrypted
payloads match the reference's, and saving writes the identical bytes."""

import json
import os
import struct

import numpy as np
import pytest

from paper_2506_19693_b200 import model_io
from paper_2506_19693_b200.he_errors import SerializationError


@pytest.fixture(scope="module")
def rbot_gold(golden_dir):
    return np.load(os.path.join(golden_dir, "ref_rbot_n512.npz"))


class _Params:
    def __init__(self, digest):
        self._d = digest

    def digest(self):
        return self._d


class _RawBackend:
    def serialize_cipher(self, cv):
        return cv

    def deserialize_cipher(self, blob):
        if blob[:4] != b"RBCT":
            raise SerializationError("bad ciphertext magic")
        return bytes(blob)


class _Custodian:
    def __init__(self, digest):
        self.params = _Params(digest)
        self.backend = _RawBackend()


def _blob(rbot_gold):
    return rbot_gold["rbot"].tobytes()


def test_container_round_trip(rbot_gold):
    blob = _blob(rbot_gold)
    cust = _Custodian(blob[16:48])
    rec = model_io.load_model(blob, cust)
    assert (rec.r, rec.c) == struct.unpack("<4sIII", blob[:16])[2:]
    assert [b.kind for b in rec.blocks] == ["RE", "CE"]
    assert [(b.in_dim, b.hidden_dim, b.out_dim) for b in rec.blocks] == [(4, 4, 2), (4, 4, 2)]
    assert rec.meta["arch"] == {"input_dim": 4, "hidden": [4, 4], "classes": 2}
    assert all(len(p) > 24 for b in rec.blocks for p in b.payloads)
    assert model_io.save_model(rec, cust) == blob


@pytest.mark.parametrize("case", ["magic", "version", "digest", "header", "blob", "kind"])
def test_container_errors(rbot_gold, case):
    blob = bytearray(_blob(rbot_gold))
    cust = _Custodian(bytes(blob[16:48]))
    if case == "magic":
        blob[:4] = b"XXXX"
    elif case == "version":
        blob[4:8] = struct.pack("<I", 2)
    elif case == "digest":
        cust = _Custodian(b"\0" * 32)
    elif case == "header":
        blob = blob[:10]
    elif case == "blob":
        blob = blob[:-100]
    else:
        (n_meta,) = struct.unpack("<I", blob[48:52])
        blob[52 + n_meta + 4] = 9  # first block's kind code
    with pytest.raises(SerializationError):
        model_io.load_model(bytes(blob), cust)


def test_meta_is_sorted_json(rbot_gold):
    blob = _blob(rbot_gold)
    (n_meta,) = struct.unpack("<I", blob[48:52])
    raw = blob[52:52 + n_meta]
    assert json.dumps(json.loads(raw), sort_keys=True).encode() == raw


@pytest.mark.gpu
def test_reference_model_loads_on_b200(rbot_gold):
    """A model saved by the reference (CPU CkksBackend) loads on the B200:
    same decrypted weights/velocities, and saving writes the same bytes."""
    from paper_2506_19693_b200.backend import load_custodian

    cust = load_custodian(rbot_gold["rbky"].tobytes())
    blob = _blob(rbot_gold)
    rec = model_io.load_model(blob, cust)
    dec = np.stack([cust.decrypt(cv).values for b in rec.blocks for cv in b.payloads])
    np.testing.assert_allclose(dec, rbot_gold["dec"], rtol=0, atol=1e-9)
    assert model_io.save_model(rec, cust) == blob
