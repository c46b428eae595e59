"""A recorded training step as one CUDA graph (the config-1 step is host-bound:
~470 small launches issued from Python take longer than the kernels run).

GraphedStep captures everything the step does on the device — the batched
plaintext encodes, the encryptions (device Philox sampler), every batched
HMult / rotation / add and the update — and replays it with one launch; the
debug refreshes, which decrypt to the host and re-encrypt (ckks/backend.py:
195-206), run eagerly after the replay, in program order.  The step's inputs
are the setup ciphertexts (weights, velocities) held in static device tensors;
outputs are the refreshed weights.  Encodes are not cached across replays: the
graph re-encodes every plaintext each time it runs, as a new step would.
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
        B.H2D_KEEPALIVE = self.keepalive
        try:
            with torch.cuda.graph(self.graph):
                self.out_env = executor.run(dict(self.static_env), only_after_setup=True,
                                            defer_refresh=True)
        finally:
            B.H2D_KEEPALIVE = None
        self.deferred = list(executor.deferred)
        be._enc_cache.clear()  # entries made during capture live in the graph's pool
        torch.cuda.synchronize()

    def step(self) -> dict:
        """Replay the captured step, then its refreshes; returns the live env."""
        self.graph.replay()
        env = dict(self.out_env)
        self.ex.deferred = list(self.deferred)
        return self.ex.finish_deferred(env)


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
