"""A recorded training step as one CUDA graph (the config-1 step is host-bound:
~470 small launches issued from Python take longer than the kernels run).

GraphedStep captures everything the step does on the device — the batched
plaintext encodes, the encryptions (device Philox sampler), every batched
HMult / rotation / add and the update — and replays it with one launch; the
debug refreshes, which decrypt to the host and re-encrypt (ckks/backend.py:
195-206), run eagerly after the replay, in program order.  The step's inputs
are the setup ciphertexts (weights, velocities) held in static device tensors;
outputs are the refreshed weights.

What a replay recomputes and what it reuses:
  * encryption randomness is FRESH per replay: every in-graph encryption
    draws its Philox stream from a key uploaded out of a pinned staging
    tensor; before each replay those tensors are rewritten with the keys of
    the serials this replay owns (the captured serials + replay index x the
    step's serial span), the eager refreshes use the same offset, and the
    backend's serial counter advances past them — no nonce is ever reused;
  * the plaintext encodes run in the graph every replay (FFT, rounding,
    residues, NTT: nothing is cached), from the recorded step's slot values —
    the plaintext inputs are those of the recorded minibatch.  Training on a
    new minibatch needs its own capture (or its values written into the
    staging tensors tagged by backend._h2d), so the replays are benchmark
    repetitions of one step with fresh randomness, not a data loader.
"""

from __future__ import annotations

import torch

from . import backend as B
from .backend import GpuCiphertext


class GraphedStep:
    def __init__(self, executor, setup_env: dict, warmup: int = 2):
        self.ex = executor
        be = executor.be
        self.be = be
        if getattr(be, "sampler", "philox") != "philox":
            raise ValueError("GraphedStep needs the device (philox) sampler: numpy-sampled "
                             "encryptions upload pageable host arrays that a graph cannot refresh")
        self.static_env = {k: GpuCiphertext(getattr(v, "payload", v).data.clone(),
                                            getattr(v, "payload", v).level)
                           for k, v in setup_env.items()}
        for _ in range(warmup):  # caches (keys, tables, FFT plans) filled eagerly
            be._enc_cache.clear()
            executor.run(dict(self.static_env), only_after_setup=True)
        torch.cuda.synchronize()
        be._enc_cache.clear()  # the graph must contain the step's own encodes
        self.graph = torch.cuda.CUDAGraph()
        self.keepalive: list = []
        executor.serial_offset = 0
        B.H2D_KEEPALIVE = self.keepalive
        try:
            with torch.cuda.graph(self.graph):
                self.out_env = executor.run(dict(self.static_env), only_after_setup=True,
                                            defer_refresh=True)
        finally:
            B.H2D_KEEPALIVE = None
        self.deferred = list(executor.deferred)
        self.seed_uploads = [(tag[1], pinned) for tag, pinned in self.keepalive
                             if isinstance(tag, tuple) and tag[0] == "seeds"]
        self.span = executor.serials_used  # serials one step may use
        self.replays = 0
        self.last_offset = 0
        self.done = None  # event: the previous replay has read its staging tensors
        be._enc_cache.clear()  # entries made during capture live in the graph's pool
        torch.cuda.synchronize()

    def step(self) -> dict:
        """Replay the captured step with fresh encryption randomness, then its
        refreshes; returns the live env."""
        self.replays += 1
        offset = self.last_offset = self.replays * self.span
        if self.done is not None:
            self.done.synchronize()  # staging tensors are free to rewrite
        for serials, pinned in self.seed_uploads:
            pinned.copy_(torch.from_numpy(
                self.be.encryption_seeds([sr + offset for sr in serials])))
        self.graph.replay()
        self.done = torch.cuda.Event()
        self.done.record()
        env = dict(self.out_env)
        self.ex.deferred = list(self.deferred)
        self.ex.serial_offset = offset
        try:
            return self.ex.finish_deferred(env)
        finally:
            import itertools

            self.be._serials = itertools.count(self.ex.serials_used + offset)
            self.ex.serial_offset = 0


def eager_equivalent(gs: GraphedStep) -> dict:
    """The eager executor's run of the step the last replay computed (same
    serial offset, so the same encryption randomness): for bit-identity checks."""
    ex = gs.ex
    ex.serial_offset = gs.last_offset
    try:
        gs.be._enc_cache.clear()
        return ex.run(dict(gs.static_env), only_after_setup=True)
    finally:
        ex.serial_offset = 0


class GraphedCall:
    """fn(*static_inputs) captured once and replayed: for fixed-shape device
    pipelines such as one bootstrapping (bootstrap.Bootstrapper via
    backend.bootstrap_ct).  Inputs are copied into static tensors with load()."""

    def __init__(self, fn, *inputs, warmup: int = 2):
        self.static_in = [x.clone() for x in inputs]
        for _ in range(warmup):
            fn(*self.static_in)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        self.keepalive: list = []
        B.H2D_KEEPALIVE = self.keepalive
        try:
            with torch.cuda.graph(self.graph):
                self.out = fn(*self.static_in)
        finally:
            B.H2D_KEEPALIVE = None
        torch.cuda.synchronize()

    def load(self, *inputs) -> None:
        for dst, src in zip(self.static_in, inputs):
            dst.copy_(src)

    def __call__(self):
        self.graph.replay()
        return self.out
