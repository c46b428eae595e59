"""Data-parallel training step: the mini-batch's samples are
sharded across ranks, one process per GPU.

``nn.train_iteration`` (/root/reference/pkg/src/ciphermlp/nn.py:344-404) runs
one independent pipeline per sample (nn.py:363-372) and folds the per-sample
gradients into ``acc`` with ``ev.add`` (nn.py:373-381); only the update and
refresh (nn.py:383-401) read the folded sums.  Over a recorded program
(replay.Program) this module derives, statically and identically on every rank:

* the sample set each value depends on (sample s = the ``encs_per_sample``
  encryptions of its inputs, in program order);
* for rank r owning samples O_r: ops depending on no sample run everywhere
  (replicated), ops depending on one sample run on its owner, and the
  ``add_ct`` ops that join disjoint sample sets (the acc chain) become rank-local
  partial sums (an operand with no owned sample is simply absent);
* before the first op that reads a multi-sample value as anything but such a
  join, one exact residue all-reduce (dist.allreduce_residues: int64 SUM then
  ``mod p`` on the device); from there on the value, and everything computed
  from it, is replicated.

Modular addition is associative, so sum_r(partial_r) mod q equals the
sequential chain bit for bit; encryption and refresh serials are the ones the
single-process program would use (WaveExecutor._plan), so the replicated update
and refresh produce the same ciphertexts on every rank and the same ones as
one GPU.  No other exchange exists on this path.
"""

from __future__ import annotations

import collections
import itertools

import numpy as np
import torch

from . import dist as hdist
from .backend import GpuCiphertext
from .executor import WaveExecutor, _inputs


def _out(op):
    return op[2] if op[0] == "ew" else op[1]


class ShardPlan:
    """Static partition of a program across `world` ranks (pure host logic)."""

    def __init__(self, ops, n_setup: int, encs_per_sample: int, world: int):
        self.world = world
        enc_ids = [i for i, op in enumerate(ops) if op[0] == "enc" and i >= n_setup]
        if encs_per_sample < 1 or len(enc_ids) % encs_per_sample:
            raise ValueError("sample encryptions do not divide into encs_per_sample groups")
        self.n_samples = len(enc_ids) // encs_per_sample
        if self.n_samples < world:
            raise ValueError(f"{self.n_samples} samples cannot feed {world} ranks")
        sample_of_enc = {i: k // encs_per_sample for k, i in enumerate(enc_ids)}
        self.owner = {}
        for r in range(world):
            for s in hdist.shard(self.n_samples, r, world):
                self.owner[s] = r
        deps = {}        # value id -> frozenset of samples (empty: replicated)
        self.kind = {}   # op index -> "rep" | ("own", rank) | "join"
        self.join_args = {}
        self.reduce_before = collections.defaultdict(list)  # op index -> [value ids]
        is_global = set()
        for i, op in enumerate(ops):
            tag = op[0]
            ins = _inputs(op)
            if tag == "enc":
                d = frozenset([sample_of_enc[i]]) if i in sample_of_enc else frozenset()
            else:
                sets = [deps[x] for x in ins]
                d = frozenset().union(*sets)
            multi = len(d) > 1
            if multi and tag == "ew" and op[1] == "add_ct" and not (sets[0] & sets[1]) \
                    and not any(x in is_global for x in ins):
                self.kind[i] = "join"
                self.join_args[i] = (op[3], op[4])
            elif multi:
                # a folded sum read by the update: reduce it once, then replicate
                for x in ins:
                    if len(deps[x]) > 1 and x not in is_global:
                        self.reduce_before[i].append(x)
                        is_global.add(x)
                    elif len(deps[x]) == 1:
                        raise ValueError(f"op {i} mixes a folded sum with one sample's value")
                d = frozenset()
                self.kind[i] = "rep"
            elif len(d) == 1:
                self.kind[i] = ("own", self.owner[next(iter(d))])
            else:
                self.kind[i] = "rep"
            deps[_out(op)] = d
        self.deps = deps
        self.reduced = sorted(is_global)

    def present(self, value_deps, rank) -> bool:
        return any(self.owner[s] == rank for s in value_deps)


class DataParallelExecutor(WaveExecutor):
    """WaveExecutor over this rank's share of the program.  `allreduce(x, limbs)`
    defaults to dist.allreduce_residues on the current process group."""

    rewrite_sums = False  # the fold's add_ct joins are the sharding's exchange points

    def __init__(self, program, custodian, encs_per_sample: int, rank: int = None,
                 world: int = None, allreduce=None):
        super().__init__(program, custodian)
        r, w = hdist.world()
        self.rank = r if rank is None else rank
        self.world_size = w if world is None else world
        self.plan = ShardPlan(program.ops, program.n_setup, encs_per_sample, self.world_size)
        self._allreduce = allreduce or self._default_allreduce
        self.exchanged_bytes = 0

    def _default_allreduce(self, x, limbs):
        return hdist.allreduce_residues(x, lambda t: self.be.chain.reduce(t, limbs))

    def _zero(self, vid):
        lvl = self.level_of[vid]
        return GpuCiphertext(torch.zeros(2, self.be._limbs(lvl), self.be.n, dtype=torch.uint64,
                                         device=self.be.device), lvl)

    def run(self, env=None, only_after_setup: bool = False) -> dict:
        be = self.be
        ops = self.prog.ops
        plan = self.plan
        rank = self.rank
        env = {} if env is None else {k: getattr(v, "payload", v) for k, v in env.items()}
        keep = self.prog.keep
        last = self.prog._last_use
        slots = be.params.slot_count
        pts = self.prog.plaintexts

        def pvals(i):
            v = np.zeros(slots)
            v[: pts.shape[1]] = pts[i]
            return v

        def runs(i):  # ops this rank executes (joins: only when both operands are here)
            k = plan.kind[i]
            if k == "join":
                a, b = plan.join_args[i]
                return plan.present(plan.deps[a], rank) and plan.present(plan.deps[b], rank)
            return k == "rep" or (isinstance(k, tuple) and k[1] == rank)

        self._pre_encode(pvals, self.n_setup if only_after_setup else 0, runs)
        for wave in self.waves:
            if only_after_setup:
                wave = [i for i in wave if i >= self.n_setup]
            todo = []
            for i in wave:
                if i in self.fused_adds:
                    continue  # produced by its rotation (WaveExecutor._plan_fusion)
                k = plan.kind[i]
                if k == "rep" or (isinstance(k, tuple) and k[1] == rank):
                    todo.append(i)
                elif k == "join":
                    a, b = plan.join_args[i]
                    ha = plan.present(plan.deps[a], rank)
                    hb = plan.present(plan.deps[b], rank)
                    if ha and hb:
                        todo.append(i)
                    elif ha or hb:
                        # the join's partial sum on this rank is the one operand
                        # present, at the join's level (add_ct adjusts operands of
                        # different levels, backend.py:94-112): every rank's
                        # partial then has the same limb count for the all-reduce
                        src = env[a if ha else b]
                        lvl = self.level_of[ops[i][2]]
                        if src.level != lvl:
                            src = GpuCiphertext(be._adjust_data(src.data, src.level, lvl), lvl)
                        env[ops[i][2]] = src
            # all-reduces first, in a rank-independent order
            for i in sorted(todo):
                for vid in plan.reduce_before.get(i, ()):
                    ct = env.get(vid) if plan.present(plan.deps[vid], rank) else None
                    if ct is None:
                        ct = self._zero(vid)
                    limbs = be._limbs(ct.level)
                    self.exchanged_bytes += ct.data.numel() * 8
                    env[vid] = GpuCiphertext(self._allreduce(ct.data.contiguous(), limbs),
                                             ct.level)
            groups = collections.defaultdict(list)
            for i in todo:
                op = ops[i]
                tag = op[0]
                if tag == "enc":
                    groups[("enc",)].append(i)
                elif tag == "ew":
                    kind, _, a, b = op[1], op[2], op[3], op[4]
                    la = env[a].level
                    if kind.endswith("_ct"):
                        groups[(kind, la, env[b].level)].append(i)
                    else:
                        groups[(kind, la, b)].append(i)
                elif tag == "rot":
                    groups[("rot", env[op[2]].level, op[3] % slots, i in self.fuse)].append(i)
                else:
                    groups[("bs", i)].append(i)
            for key, idx in groups.items():
                self._run_group(key, idx, env, pvals)
            for i in wave:
                for ref in _inputs(ops[i]):
                    if last.get(ref) == i and ref not in keep:
                        env.pop(ref, None)
        be._serials = itertools.count(self.serials_used)
        return env
