"""Deferred execution of live HE-API calls (on the real drop-in path).

With ``deferred=True`` (backend option, e.g. ``plugin.install(deferred=True)``)
the B200 backend does not launch anything when the reference layer code calls
encrypt / elementwise / rotate / bootstrap: each hook appends the call to a
program and returns a ``LazyPayload``.  The program is executed the first time
a result must leave the device — ``decrypt``, ``serialize_cipher`` — or on an
explicit ``backend.flush()``, by the same ``executor.WaveExecutor`` the
recorded-trace benchmarks use: dependency waves, ops of a wave with the same
signature as ONE batched launch sequence (the B samples of
``nn.train_iteration``, nn.py:363-382, share every rotation-key read and
plaintext), rotate-and-accumulate fusion, and deferred batched refreshes.

Semantics are those of eager execution, bit for bit: every recorded
encryption / refresh keeps the RNG serial the eager hook would have drawn
(``_serials`` is advanced at record time exactly as the eager hooks do), debug
refreshes keep program order (their eps draws), and integer ops are exact, so
the batched results equal sequential ones (tests/test_gpu_dropin.py).  The
level / depth / keyset checks of the HE API still run at call time in the
base class; only the arithmetic is deferred.

Pipelined flushes (``deferred_async=True``): ``flush()`` hands the recorded
program to one worker thread that plans it and issues its launches, and
returns at once, so the layer code records step t+1 while step t's kernels
are still being issued and run (the launch queue holds well under one step of
a bootstrapped training configuration, so a synchronous flush leaves the GPU
idle for the whole recording of the next step).  Programs run in flush order;
a value from a pending program is an *input* of the next one, read when that
program starts.  ``resolve`` (decrypt / serialize) and ``wait()`` join the
worker.  The live RNG serial counter belongs to the recording thread only.
"""

from __future__ import annotations

import concurrent.futures
import itertools
import types
import weakref

import numpy as np

from .backend import GpuCiphertext


class LazyPayload:
    """Placeholder payload of a deferred op; ``value`` is the GpuCiphertext once
    its program has run."""

    __slots__ = ("vid", "level", "value", "__weakref__")

    def __init__(self, vid: int, level: int):
        self.vid = vid
        self.level = level
        self.value = None


class _Program:
    """The minimal replay.Program surface WaveExecutor reads."""

    def __init__(self, ops, plaintexts, outputs):
        self.ops = ops
        self.plaintexts = plaintexts
        self.outputs = list(outputs)
        self.n_setup = 0
        self.carry = set()
        last = {}
        for i, op in enumerate(ops):
            for ref in _inputs(op):
                last[ref] = i
        self._last_use = last

    @property
    def keep(self) -> set:
        return set(self.outputs)


def _inputs(op):
    tag = op[0]
    if tag == "ew":
        return [op[3]] + ([op[4]] if op[1].endswith("_ct") else [])
    if tag in ("rot", "bs"):
        return [op[2]]
    return []


class Recorder:
    """Per-backend recording state."""

    def __init__(self, backend, max_ops: int = 250_000, max_group: int = None,
                 pipelined: bool = False):
        self.be = backend
        self.max_ops = max_ops
        self.max_group = max_group  # WaveExecutor sub-batch bound (peak memory)
        self.pipelined = pipelined
        self._worker = None
        self._pending = []
        self._ids = itertools.count()
        self._reset()

    def _reset(self):
        self.ops = []
        self.serials = {}            # op index -> RNG serial of an enc / bs
        self.pts: dict = {}          # plaintext bytes -> index
        self.pt_rows = []
        self.inputs = {}             # vid -> GpuCiphertext (materialized operands)
        self.input_of = {}           # id(GpuCiphertext) -> vid
        self.lazy = weakref.WeakValueDictionary()  # vid -> LazyPayload still referenced

    # -- operands -------------------------------------------------------------
    def operand(self, payload) -> int:
        if isinstance(payload, LazyPayload):
            if payload.value is not None:  # ran in an earlier flush
                payload = payload.value
            elif payload.vid in self.lazy:  # recorded in this program
                return payload.vid
            else:  # produced by a pending (pipelined) program: an input, read at run time
                self.inputs[payload.vid] = payload
                return payload.vid
        key = id(payload)
        vid = self.input_of.get(key)
        if vid is None:
            vid = next(self._ids)
            self.input_of[key] = vid
            self.inputs[vid] = payload
        return vid

    def plaintext(self, values) -> int:
        v = np.ascontiguousarray(values, dtype=np.float64)
        key = v.tobytes()
        idx = self.pts.get(key)
        if idx is None:
            idx = self.pts[key] = len(self.pt_rows)
            self.pt_rows.append(v)
        return idx

    def new(self, level: int) -> LazyPayload:
        lp = LazyPayload(next(self._ids), level)
        self.lazy[lp.vid] = lp
        return lp

    # -- recording --------------------------------------------------------------
    def record(self, op, level: int, serial=None) -> LazyPayload:
        out = self.new(level)
        op = tuple(x if x is not None else out.vid for x in op)
        if serial is not None:
            self.serials[len(self.ops)] = serial
        self.ops.append(op)
        if len(self.ops) >= self.max_ops:
            self.flush()
        return out

    # -- execution --------------------------------------------------------------
    def flush(self, on_issued=None) -> None:
        """Run (pipelined: submit) everything recorded so far.  on_issued(): called
        on the issuing thread right after the program's last launch (e.g. to
        record a CUDA event at a training-step boundary)."""
        if not self.ops:
            if on_issued is not None:
                if self.pipelined and self._pending:
                    self._submit(on_issued)
                else:
                    on_issued()
            return
        snap = (self.ops, self.serials, self.inputs, dict(self.lazy),
                np.stack(self.pt_rows) if self.pt_rows else np.zeros((0, 1)))
        self._reset()
        if not self.pipelined:
            self._run(snap, restore_serials=True)
            if on_issued is not None:
                on_issued()
            return

        def job():
            self._run(snap, restore_serials=False)
            if on_issued is not None:
                on_issued()

        self._submit(job)

    def _submit(self, fn) -> None:
        if self._worker is None:
            self._worker = concurrent.futures.ThreadPoolExecutor(
                max_workers=1, thread_name_prefix="ckb-flush")
        dev = getattr(self.be, "device", None)

        def job():
            import torch

            if dev is not None and torch.device(dev).type == "cuda":
                torch.cuda.set_device(dev)  # the recording thread's device (one per rank)
            fn()

        self._pending.append(self._worker.submit(job))

    def wait(self) -> None:
        """Join every pending pipelined program (re-raises its error)."""
        pending, self._pending = self._pending, []
        for f in pending:
            f.result()

    def _run(self, snap, restore_serials: bool) -> None:
        from .executor import WaveExecutor

        be = self.be
        ops, serials, inputs, live, pts = snap
        # values of earlier (pipelined) programs have been produced by now:
        # programs run in flush order on one thread
        vals = {}
        for k, v in inputs.items():
            if isinstance(v, LazyPayload):
                if v.value is None:
                    raise RuntimeError("deferred input was not produced by an earlier program")
                v = v.value
            vals[k] = v
        prog = _Program(ops, pts, [v for v in live if v not in inputs])
        view = types.SimpleNamespace(backend=be)
        ex = WaveExecutor(prog, view, max_group=self.max_group,
                          inputs={k: v.level for k, v in vals.items()})
        ex.serial_of = dict(serials)
        if restore_serials:
            saved = be._serials
            try:
                env = ex.run(dict(vals))
            finally:
                be._serials = saved  # the live counter already advanced at record time
        else:  # the recording thread owns the live counter: leave it alone
            env = ex.run(dict(vals), update_serials=False)
        for vid, lp in live.items():
            val = env.get(vid)
            if val is not None:
                lp.value = val

    def resolve(self, payload) -> GpuCiphertext:
        if isinstance(payload, LazyPayload):
            if payload.value is None:
                self.flush()
                self.wait()
            if payload.value is None:
                raise RuntimeError("deferred value was not produced by its program")
            return payload.value
        return payload
