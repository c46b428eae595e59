"""Wavefront-batched execution of a recorded HE program.

``nn.train_iteration`` (/root/reference/pkg/src/ciphermlp/nn.py:344-404) runs
B independent per-sample pipelines (nn.py:363-382) and then the update.  Issued
one HE call at a time, each call is a handful of small kernels on ~0.5 MB
ciphertexts (config 1), so the step is launch- and host-bound and every
rotation re-reads its key.  HE ops are pure functions of their operands, so
the program (replay.Program: the exact call sequence the layer code makes) can
be executed in dependency waves: all ops whose inputs are ready form a wave,
and ops of a wave that share a signature — (kind, operand levels, rotation
step, plaintext) — run as ONE batched launch sequence over stacked operands
(one key read per rotation group, one plaintext per mul_pt group).

Results are identical to sequential execution: every integer op is exact,
encryption randomness is drawn from the serial each call would have had in
program order (pre-assigned here), and refreshes run in program order.
"""

from __future__ import annotations

import collections

import numpy as np
import torch

from .backend import GpuCiphertext


class WaveExecutor:
    def __init__(self, program, custodian, max_group: int = None, inputs: dict = None):
        """max_group: split a wave's same-signature group into sub-batches of at
        most this many ops (bounds the temporaries of very wide steps; results
        are unchanged — every op is computed independently)."""
        self.prog = program
        self.cust = custodian
        self.be = custodian.backend
        self.max_group = max_group
        # values the program reads but no op produces (deferred.Recorder: the
        # already-materialized operands), id -> level
        self.inputs = dict(inputs or {})
        # added to every serial the plan assigns: a replayed step (graphs.
        # GraphedStep) draws fresh encryption randomness per replay
        self.serial_offset = 0
        self._plan()

    # -- planning ------------------------------------------------------------
    def _plan(self):
        """Serials (as the HE API would assign them) and dependency waves."""
        ops = self.prog.ops
        be = self.be
        ser = {}
        counter = 0
        depth = {}
        waves = collections.defaultdict(list)
        level = dict(self.inputs)
        self._last_bs_depth = 0
        top = be.params.level
        rl = be.params.refresh_level
        self.n_setup = self.prog.n_setup
        self._plan_fusion()
        self._plan_sums()

        for i, op in enumerate(ops):
            tag = op[0]
            if i in self.absorbed:  # inner add of a summation tree (_plan_sums)
                counter += 1
                level[op[2]] = min(level[op[3]], level[op[4]])  # bookkeeping only
                continue
            if tag == "enc":
                ser[i] = counter + 1          # api.py:225 then backend.py:174
                counter += 2
                out, ins, lvl = op[1], [], top
            elif tag == "ew":
                kind, out, a, b = op[1], op[2], op[3], op[4]
                ins = self.sums.get(i) or ([a] + ([b] if kind.endswith("_ct") else []))
                lvl = min(level[x] for x in ins)
                if kind.startswith("mul"):
                    lvl -= 1
                counter += 1
            elif tag == "rot":
                out, ins = op[1], [op[2]]
                lvl = level[op[2]]
                counter += 1
            elif tag == "bs":
                out, ins = op[1], [op[2]]
                ser[i] = counter + 1          # api.py:246 then backend.py:174 (re-encrypt)
                counter += 2
                lvl = rl
            else:
                raise ValueError(tag)
            d = 1 + max((depth.get(x, 0) for x in ins), default=0)
            if tag == "bs" and not be.real_bootstrap:
                # debug refreshes keep program order (their bs_rng draws); real
                # bootstraps are deterministic and batch freely
                d = max(d, self._last_bs_depth + 1)
                self._last_bs_depth = d
            depth[out] = d
            level[out] = lvl
            waves[d].append(i)
        # real bootstraps whose outputs nothing in the step reads (the refreshed
        # weights): deferred to one final wave and run as a single batch (each
        # input is first brought to level 0, where bootstrapping starts anyway)
        if be.real_bootstrap:
            bs = [i for i, op in enumerate(ops) if op[0] == "bs" and i >= self.n_setup]
            consumed = {x for op in ops for x in _inputs(op)}
            if len(bs) > 1 and not any(ops[i][1] in consumed for i in bs):
                last_d = max(waves) + 1
                for d in list(waves):
                    waves[d] = [i for i in waves[d] if ops[i][0] != "bs"]
                    if not waves[d]:
                        del waves[d]
                waves[last_d] = bs
        self.serial_of = ser
        self.level_of = level
        self.waves = [waves[d] for d in sorted(waves)]
        self.serials_used = counter
        last = {}
        for i, op in enumerate(ops):
            if i in self.absorbed:
                continue
            for ref in self.sums.get(i) or _inputs(op):
                last[ref] = i
        self.last_use = last

    rewrite_sums = True  # the data-parallel executor keeps the fold's joins

    def _plan_sums(self):
        """Summation trees: a chain of add_ct ops whose intermediate sums have
        exactly one reader (the delta-W fold over the B samples, nn.py:373-381:
        acc = acc + dW_s) becomes ONE n-ary sum at its last add, executed as a
        log-depth tree of batched adds (modular addition is exact and
        associative, so the value is unchanged) instead of B - 1 dependent
        single-ciphertext waves.  Leaves must share one level (no adjusts)."""
        ops = self.prog.ops
        self.sums, self.absorbed = {}, set()
        if not self.rewrite_sums:
            return
        keep = self.prog.keep
        readers = collections.defaultdict(list)
        producer = {}
        for j, op in enumerate(ops):
            for x in _inputs(op):
                readers[x].append(j)
            producer[_output(op)] = j

        def is_add(j):
            op = ops[j]
            return (op[0] == "ew" and op[1] == "add_ct" and j >= self.n_setup
                    and j not in self.fused_adds)

        def internal(x, j):
            i = producer.get(x)
            return (i is not None and is_add(i) and x not in keep and readers.get(x) == [j])

        # levels of every value (no rewrite) to check the leaves
        level = dict(self.inputs)
        top, rl = self.be.params.level, self.be.params.refresh_level
        for op in ops:
            tag = op[0]
            if tag == "enc":
                level[op[1]] = top
            elif tag == "ew":
                ins = [op[3]] + ([op[4]] if op[1].endswith("_ct") else [])
                lv = min(level[x] for x in ins)
                level[op[2]] = lv - 1 if op[1].startswith("mul") else lv
            elif tag == "rot":
                level[op[1]] = level[op[2]]
            else:
                level[op[1]] = rl
        for j in range(len(ops)):
            if not is_add(j) or any(internal(_output(ops[j]), r)
                                    for r in readers.get(_output(ops[j]), [])):
                continue  # not a root (its sum feeds the next add of a chain)
            leaves, inner, stack = [], [], [j]
            while stack:
                k = stack.pop()
                for x in (ops[k][3], ops[k][4]):
                    if internal(x, k):
                        inner.append(producer[x])
                        stack.append(producer[x])
                    else:
                        leaves.append(x)
            if len(leaves) >= 3 and len({level[x] for x in leaves}) == 1:
                self.sums[j] = leaves
                self.absorbed.update(inner)

    def _plan_fusion(self):
        """Rotate-and-accumulate pairs: rot i (o = rotate(s, k)) whose result's
        only reader is add_ct j = s + o (either operand order) — every rotation
        of the recorded training steps (the log-depth sums of packing.py:193-208
        and linalg.py:60-82).  Op i then produces j's output directly
        (backend._hrot(accumulate=True): the add rides in the ModDown combine)
        and j is skipped; modular addition is exact, so values are unchanged."""
        ops = self.prog.ops
        readers = collections.defaultdict(list)
        for j, op in enumerate(ops):
            for x in _inputs(op):
                readers[x].append(j)
        keep = self.prog.keep
        self.fuse = {}
        for i, op in enumerate(ops):
            if op[0] != "rot":
                continue
            o, src = op[1], op[2]
            rd = readers.get(o, [])
            if o in keep or len(rd) != 1:
                continue
            j = rd[0]
            add = ops[j]
            if add[0] == "ew" and add[1] == "add_ct" and {add[3], add[4]} == {o, src}:
                self.fuse[i] = j
        self.fused_adds = set(self.fuse.values())

    # -- execution -----------------------------------------------------------
    def run(self, env=None, only_after_setup: bool = False, defer_refresh: bool = False,
            update_serials: bool = True) -> dict:
        """Execute the program; returns id -> GpuCiphertext for live values.
        With only_after_setup, ops before program.n_setup must already be in env.
        defer_refresh: debug refreshes (a host round trip each) are not run but
        listed in self.deferred, to be finished by finish_deferred(env); used by
        graphs.GraphedStep to capture everything else in one CUDA graph."""
        be = self.be
        ops = self.prog.ops
        env = {} if env is None else {k: getattr(v, "payload", v) for k, v in env.items()}
        keep = self.prog.keep
        last = self.last_use
        slots = be.params.slot_count
        pts = self.prog.plaintexts

        def pvals(i):
            v = np.zeros(slots)
            v[: pts.shape[1]] = pts[i]
            return v

        self._pre_encode(pvals, self.n_setup if only_after_setup else 0)
        self.deferred = []
        self._pvals = pvals
        deferring = defer_refresh and not be.real_bootstrap
        for wave in self.waves:
            if only_after_setup:
                wave = [i for i in wave if i >= self.n_setup]
                if not wave:
                    continue
            if deferring:
                bs = [i for i in wave if ops[i][0] == "bs"]
                self.deferred.extend(bs)
                wave = [i for i in wave if ops[i][0] != "bs"]
                for i in wave:  # nothing may consume a deferred refresh
                    if any(ops[j][1] in _inputs(ops[i]) for j in self.deferred):
                        raise ValueError("an op reads a deferred refresh output")
            groups = collections.defaultdict(list)
            for i in wave:
                op = ops[i]
                tag = op[0]
                if i in self.fused_adds:
                    continue  # produced by its rotation (_plan_fusion)
                if i in self.sums:  # n-ary summation tree (_plan_sums)
                    leaves = self.sums[i]
                    groups[("sum", env[leaves[0]].level, len(leaves))].append(i)
                    continue
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
                elif be.real_bootstrap:  # one batched bootstrapping
                    groups[("bs", "batch")].append(i)
                else:
                    groups[("bs", i)].append(i)
            for key, idx in groups.items():
                step = self.max_group or len(idx)
                for lo in range(0, len(idx), step):
                    self._run_group(key, idx[lo:lo + step], env, pvals)
            for i in wave:
                for ref in self.sums.get(i) or _inputs(ops[i]):
                    if last.get(ref) == i and ref not in keep:
                        env.pop(ref, None)
        # leave the backend's serial counter where sequential execution would
        # (not for a pipelined deferred program: the recording thread owns it)
        if update_serials:
            import itertools

            be._serials = itertools.count(self.serials_used + self.serial_offset)
        return env

    def finish_deferred(self, env: dict) -> dict:
        """Run the debug refreshes run(defer_refresh=True) skipped — together:
        one batched decrypt per level (one device->host copy), the eps noise
        drawn in program order, one batched re-encryption with each refresh's
        own serial — so the results equal refreshing one at a time."""
        be = self.be
        ops = self.prog.ops
        keep = self.prog.keep
        last = self.last_use
        order = sorted(self.deferred)
        if not order:
            return env
        values = {}
        by_level: dict = {}
        for i in order:
            by_level.setdefault(env[ops[i][2]].level, []).append(i)
        for lvl, idx in by_level.items():
            dec = be._decrypt_values_batch(torch.stack([env[ops[i][2]].data for i in idx]), lvl)
            for j, i in enumerate(idx):
                values[i] = dec[j]
        for i in order:  # backend.py:195-206: + U(-eps, eps), in program order
            if be.bootstrap_eps > 0.0:
                values[i] = values[i] + be._bs_rng.uniform(-be.bootstrap_eps, be.bootstrap_eps,
                                                           values[i].shape[0])
        rl = be.params.refresh_level
        data = be._encrypt_batch([values[i] for i in order], rl,
                                 [self.serial_of[i] + self.serial_offset for i in order])
        for j, i in enumerate(order):
            env[ops[i][1]] = GpuCiphertext(data[j], rl)
            for ref in _inputs(ops[i]):
                if last.get(ref) == i and ref not in keep:
                    env.pop(ref, None)
        return env

    def _pre_encode(self, pvals, start: int, runs=None) -> None:
        """Every plaintext the program will encode, batched per (level, NTT form)
        before the first wave (backend.encode_many); the per-op encodes then hit
        the cache.  Levels are the static ones of _plan."""
        ops = self.prog.ops
        top = self.be.params.level
        items = []
        for i in range(start, len(ops)):
            op = ops[i]
            if runs is not None and not runs(i):
                continue
            if op[0] == "enc":
                items.append((pvals(op[2]), top, False))
            elif op[0] == "ew" and not op[1].endswith("_ct"):
                kind, a, pid = op[1], op[3], op[4]
                v = pvals(pid)
                items.append((-v if kind.startswith("sub") else v, self.level_of[a], True))
        if items and hasattr(self.be, "encode_many"):
            self.be.encode_many(items)

    def _stack(self, items):
        if len(items) == 1:
            return items[0].unsqueeze(0)
        return torch.stack(items)

    def _run_group(self, key, idx, env, pvals):
        be = self.be
        ch = be.chain
        ops = self.prog.ops
        tag = key[0]
        if tag == "enc":
            top = be.params.level
            data = be._encrypt_batch([pvals(ops[i][2]) for i in idx], top,
                                     [self.serial_of[i] + self.serial_offset for i in idx])
            for j, i in enumerate(idx):
                env[ops[i][1]] = GpuCiphertext(data[j], top)
            return
        if tag == "bs":
            if be.real_bootstrap:  # homomorphic bootstrapping (bootstrap.py), batched
                ins = [env[ops[i][2]] for i in idx]
                lvl = min(c.level for c in ins)
                if lvl > 0 or any(c.level != lvl for c in ins):
                    lvl = 0  # bootstrapping starts from level 0 anyway
                    datas = [c.data if c.level == 0 else be._adjust_data(c.data, c.level, 0)
                             for c in ins]
                else:
                    datas = [c.data for c in ins]
                out = be.bootstrap_batch(self._stack(datas), lvl)
                rl = be.params.refresh_level
                for j, i in enumerate(idx):
                    env[ops[i][1]] = GpuCiphertext(out[j], rl)
                return
            i = idx[0]
            src = env[ops[i][2]]
            values = be._decrypt_values(src)
            if be.bootstrap_eps > 0.0:
                values = values + be._bs_rng.uniform(-be.bootstrap_eps, be.bootstrap_eps,
                                                     values.shape[0])
            rl = be.params.refresh_level
            env[ops[i][1]] = GpuCiphertext(
                be._encrypt_batch([values], rl, [self.serial_of[i] + self.serial_offset])[0], rl)
            return
        if tag == "sum":  # log-depth tree of batched adds over every root's leaves
            _, lvl, _k = key
            m = be._limbs(lvl)
            x = torch.stack([torch.stack([env[v].data for v in self.sums[i]]) for i in idx])
            while x.shape[1] > 1:
                k = x.shape[1]
                h = k // 2
                y = ch.add(x[:, :h].contiguous(), x[:, h:2 * h].contiguous(), m)
                x = torch.cat([y, x[:, 2 * h:]], dim=1) if k % 2 else y
            for j, i in enumerate(idx):
                env[ops[i][2]] = GpuCiphertext(x[j, 0], lvl)
            return
        if tag == "rot":
            _, lvl, step, fused = key
            x = self._stack([env[ops[i][2]].data for i in idx])
            if step == 0:
                out = ch.add(x, x, be._limbs(lvl)) if fused else x.clone()
            else:
                g = be.galois_for_step.get(step, pow(5, step, 2 * be.n))
                out = be._hrot(x, lvl, galois=g, key=be.rotation_key(g), accumulate=fused)
            for j, i in enumerate(idx):
                dst = ops[self.fuse[i]][2] if fused else ops[i][1]
                env[dst] = GpuCiphertext(out[j], lvl)
            return
        kind = tag
        op3 = kind[:3]
        if kind.endswith("_ct"):
            _, la, lb = key
            lvl = min(la, lb)
            in_level = lvl
            a = self._stack([env[ops[i][3]].data for i in idx])
            b = self._stack([env[ops[i][4]].data for i in idx])
            if la != in_level:
                a = be._adjust_data(a, la, in_level)
            if lb != in_level:
                b = be._adjust_data(b, lb, in_level)
            m = be._limbs(in_level)
            if op3 == "add":
                out, out_level = ch.add(a, b, m), in_level
            elif op3 == "sub":
                out, out_level = ch.sub(a, b, m), in_level
            else:
                out, out_level = be._hmult(a.contiguous(), b.contiguous(), in_level), in_level - 1
        else:
            _, la, pid = key
            m = be._limbs(la)
            vals = pvals(pid)
            a = self._stack([env[ops[i][3]].data for i in idx])
            if op3 == "mul":
                pt = be._encode_rns(vals, la, ntt=True)
                out = be._rescale_data(ch.mul(a, pt, m, b_rows=m), la)
                out_level = la - 1
            else:
                pt = be._encode_rns(vals if op3 == "add" else -vals, la, ntt=True)
                pt2 = torch.zeros(2, m, be.n, dtype=pt.dtype, device=pt.device)
                pt2[0].copy_(pt)  # (c0 + pt, c1 + 0), broadcast over the batch
                out = ch.ew(0, torch.empty_like(a), a, pt2, limbs=m, b_rows=2 * m)
                out_level = la
        for j, i in enumerate(idx):
            env[ops[i][2]] = GpuCiphertext(out[j], out_level)


def _output(op):
    return op[2] if op[0] == "ew" else op[1]


def _inputs(op):
    tag = op[0]
    if tag == "ew":
        return [op[3]] + ([op[4]] if op[1].endswith("_ct") else [])
    if tag in ("rot", "bs"):
        return [op[2]]
    return []
