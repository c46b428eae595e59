"""RBOT trained-model container on the B200 backend.

The reference writes a trained model as ``RBOT`` (``ciphermlp/serialize.py:15-107``):
``<4sIII`` magic/version/grid r/grid c, the 32-byte scheme-parameter digest, a
length-prefixed JSON blob (hyperparameters, architecture, flags), then per block
``<BIIII`` kind/index/in/hidden/out and four length-prefixed RBCT ciphertexts
(layer weights, classifier weights and their velocities).  With the plugin
installed the reference's own ``save_model``/``load_model`` already run on this
backend (they only call ``backend.serialize_cipher``/``deserialize_cipher``).
This module is the same container for callers that hold the B200 backend
without the ``ciphermlp`` package — the recorded-step executors, whose
refreshed weights are plain ``CipherVector``s — so a model trained here loads
into the reference (and back) byte for byte.
"""

from __future__ import annotations

import dataclasses
import io
import json
import struct

from .he_errors import SerializationError

MODEL_MAGIC = b"RBOT"          # serialize.py:15
MODEL_VERSION = 1              # serialize.py:16
KIND_CODES = {"RE": 1, "CE": 2}  # serialize.py:18
KIND_FROM_CODE = {v: k for k, v in KIND_CODES.items()}
_HEAD = "<4sIII"
_BLOCK = "<BIIII"
PAYLOAD_NAMES = ("layer_weights", "classifier_weights", "layer_velocity",
                 "classifier_velocity")


@dataclasses.dataclass
class ModelBlock:
    """One local-loss block (nn.py:61-78): kind "RE"/"CE" and its 4 ciphertexts."""

    kind: str
    index: int
    in_dim: int
    hidden_dim: int
    out_dim: int
    payloads: tuple  # 4 CipherVectors, PAYLOAD_NAMES order

    def __post_init__(self):
        if self.kind not in KIND_CODES:
            raise SerializationError(f"unknown block kind {self.kind!r}")
        if len(self.payloads) != 4:
            raise SerializationError("a block carries exactly 4 ciphertexts")


@dataclasses.dataclass
class ModelRecord:
    """Grid shape, the JSON metadata (serialize.py:44-51) and the blocks."""

    r: int
    c: int
    meta: dict
    blocks: list


def _write_blob(out: io.BytesIO, blob: bytes) -> None:       # serialize.py:22-24
    out.write(struct.pack("<I", len(blob)))
    out.write(blob)


def _read_blob(buf: io.BytesIO) -> bytes:                    # serialize.py:27-35
    raw = buf.read(4)
    if len(raw) != 4:
        raise SerializationError("truncated container")
    (n,) = struct.unpack("<I", raw)
    blob = buf.read(n)
    if len(blob) != n:
        raise SerializationError("truncated blob")
    return blob


def _read_exact(buf: io.BytesIO, n: int, what: str) -> bytes:
    raw = buf.read(n)
    if len(raw) != n:
        raise SerializationError(f"truncated {what}")
    return raw


def save_model(record: ModelRecord, custodian) -> bytes:
    """serialize.py:38-60: same field order and encodings, JSON with sorted keys."""
    backend = custodian.backend
    out = io.BytesIO()
    out.write(struct.pack(_HEAD, MODEL_MAGIC, MODEL_VERSION, record.r, record.c))
    out.write(custodian.params.digest())
    _write_blob(out, json.dumps(record.meta, sort_keys=True).encode())
    out.write(struct.pack("<I", len(record.blocks)))
    for b in record.blocks:
        out.write(struct.pack(_BLOCK, KIND_CODES[b.kind], b.index, b.in_dim, b.hidden_dim,
                              b.out_dim))
        for cv in b.payloads:
            _write_blob(out, backend.serialize_cipher(cv))
    return out.getvalue()


def load_model(blob: bytes, custodian) -> ModelRecord:
    """serialize.py:63-107, with the same SerializationError cases."""
    buf = io.BytesIO(blob)
    head = buf.read(struct.calcsize(_HEAD))
    if len(head) != struct.calcsize(_HEAD):
        raise SerializationError("truncated model header")
    magic, version, r, c = struct.unpack(_HEAD, head)
    if magic != MODEL_MAGIC:
        raise SerializationError(f"bad model magic {magic!r}")
    if version != MODEL_VERSION:
        raise SerializationError(f"unsupported model version {version}")
    digest = buf.read(32)
    if digest != custodian.params.digest():
        raise SerializationError("model was trained under different scheme parameters")
    meta = json.loads(_read_blob(buf).decode())
    (n_blocks,) = struct.unpack("<I", _read_exact(buf, 4, "block count"))
    backend = custodian.backend
    blocks = []
    for _ in range(n_blocks):
        code, index, in_dim, hidden_dim, out_dim = struct.unpack(
            _BLOCK, _read_exact(buf, struct.calcsize(_BLOCK), "block header"))
        kind = KIND_FROM_CODE.get(code)
        if kind is None:
            raise SerializationError(f"unknown block kind code {code}")
        payloads = tuple(backend.deserialize_cipher(_read_blob(buf)) for _ in range(4))
        blocks.append(ModelBlock(kind, index, in_dim, hidden_dim, out_dim, payloads))
    return ModelRecord(r=r, c=c, meta=meta, blocks=blocks)
