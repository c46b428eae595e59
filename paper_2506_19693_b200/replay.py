"""Replay a recorded HE-API program through a KeyCustodian.

The config-1 training step is the reference's unchanged ``nn.train_iteration``
(/root/reference/pkg/src/ciphermlp/nn.py:344-404).  The reference package is
not shipped to the GPU box, so tests/golden/make_golden.py records the exact
sequence of HE-API calls that function makes (encrypt / elementwise / rotate /
bootstrap, with operand ids and plaintext vectors) and this module issues the
same calls, in the same order, against this package's HE API — the B200
backend sees precisely the workload the layer code generates.
"""

from __future__ import annotations

import json

import numpy as np

from .he_api import make_plain


class Program:
    def __init__(self, ops, plaintexts: np.ndarray, outputs, n_setup: int = 0, carry=()):
        """carry: ids a later program (the next training step) reads; kept
        alive like the outputs."""
        self.ops = ops
        self.plaintexts = plaintexts
        self.outputs = [int(o) for o in outputs]
        self.n_setup = int(n_setup)
        self.carry = {int(c) for c in carry}
        last = {}
        for i, op in enumerate(ops):
            for ref in _inputs(op):
                last[ref] = i
        self._last_use = last

    @property
    def keep(self) -> set:
        """Ids kept alive past their last use: the outputs and the carry."""
        return set(self.outputs) | self.carry

    @classmethod
    def load(cls, path: str) -> "Program":
        """The recorded step (setup ops, then one train_iteration).  Traces with
        a second iteration (ops_step2) keep the values it reads alive."""
        z = np.load(path)
        ops = json.loads(str(z["ops"]))
        carry = ()
        if "ops_step2" in z:
            ops2 = json.loads(str(z["ops_step2"]))
            defined = {_output(op) for op in ops2}
            carry = {x for op in ops2 for x in _inputs(op)} - defined
        return cls(ops, z["plaintexts"], z["outputs"], int(z["n_setup"][0]), carry)

    @classmethod
    def load_step2(cls, path: str) -> "Program":
        """The trace's second train_iteration (the steady state: weights and
        velocities refreshed to the refresh level by step 1's bootstraps) as a
        program whose "setup" is everything before it: run it with
        only_after_setup on the environment step 1 leaves."""
        z = np.load(path)
        ops = json.loads(str(z["ops"]))
        ops2 = json.loads(str(z["ops_step2"]))
        return cls(ops + ops2, z["plaintexts"], z["outputs_step2"], len(ops))

    def run(self, custodian, start: int = 0, stop: int = None, env: dict = None) -> dict:
        ev = custodian.evaluator
        slots = custodian.params.slot_count
        bits = float(custodian.params.scale_bits)
        pts = {}
        env = {} if env is None else env
        keep = self.keep
        stop = len(self.ops) if stop is None else stop

        def pt(i):
            if i not in pts:
                pts[i] = make_plain(self.plaintexts[i], slots, bits)
            return pts[i]

        for i in range(start, stop):
            op = self.ops[i]
            tag = op[0]
            if tag == "enc":
                env[op[1]] = custodian.encrypt(pt(op[2]))
            elif tag == "ew":
                kind, out, a, b = op[1], op[2], op[3], op[4]
                rhs = env[b] if kind.endswith("_ct") else pt(b)
                env[out] = ev.elementwise(kind, env[a], rhs)
            elif tag == "rot":
                env[op[1]] = ev.rotate(env[op[2]], op[3])
            elif tag == "bs":
                env[op[1]] = custodian.bootstrap(env[op[2]])
            else:
                raise ValueError(f"unknown op {tag!r}")
            for ref in _inputs(op):
                if self._last_use.get(ref) == i and ref not in keep:
                    env.pop(ref, None)
        return env


def _output(op):
    return op[2] if op[0] == "ew" else op[1]


def _inputs(op):
    tag = op[0]
    if tag == "ew":
        return [op[3]] + ([op[4]] if op[1].endswith("_ct") else [])
    if tag in ("rot", "bs"):
        return [op[2]]
    return []
