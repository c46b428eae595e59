"""Data-parallel sharding of the recorded training step (dp.ShardPlan,
SURVEY.md §8(e)) — host logic on CPU.

The plan is checked structurally on the c1/c4 traces, then exercised with a
world-size-2 gloo run of an exact stand-in semantics (every ciphertext is a
vector mod a prime; add/sub/mul are slot-wise mod q, rotation is a roll,
refresh is the identity): each rank interprets only its share, folds its
partial sums, and all-reduces exactly where the plan says.  The ranks' outputs
must equal the sequential interpretation bit for bit, which is the property
the GPU run relies on (modular addition is associative)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

Q = 2147483647  # 2^31 - 1: products of residues stay below 2^62
SLOTS = 64


def _program(golden_dir, name):
    from paper_2506_19693_b200.replay import Program

    return Program.load(os.path.join(golden_dir, name))


@pytest.mark.parametrize("name,n_samples", [("c1_trace.npz", 32), ("c4_trace.npz", 128)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_partitions_samples(golden_dir, name, n_samples, world):
    from paper_2506_19693_b200.dp import ShardPlan

    prog = _program(golden_dir, name)
    plan = ShardPlan(prog.ops, prog.n_setup, 3, world)
    assert plan.n_samples == n_samples
    owned = [0] * world
    for i, k in plan.kind.items():
        if isinstance(k, tuple):
            owned[k[1]] += 1
    # per-sample work splits evenly (samples are contiguous shards)
    assert max(owned) - min(owned) <= max(owned) // max(1, n_samples // world)
    # exactly the folded gradients (layer + classifier per block) are reduced,
    # and each is the output of a join (the nn.py:373-381 add chain)
    joins = {prog.ops[i][2] for i, k in plan.kind.items() if k == "join"}
    assert plan.reduced and set(plan.reduced) <= joins
    assert len(plan.reduced) % 2 == 0
    # the update + refresh read only reduced (replicated) values
    for i, k in plan.kind.items():
        if k == "rep" and prog.ops[i][0] == "bs":
            assert not plan.deps[prog.ops[i][2]]


def test_plan_rejects_too_few_samples(golden_dir):
    from paper_2506_19693_b200.dp import ShardPlan

    prog = _program(golden_dir, "c1_trace.npz")
    with pytest.raises(ValueError):
        ShardPlan(prog.ops, prog.n_setup, 3, 33)
    with pytest.raises(ValueError):
        ShardPlan(prog.ops, prog.n_setup, 5, 2)


def _pt(pid):
    return np.random.default_rng(1000 + pid).integers(0, Q, SLOTS, dtype=np.int64)


def _apply(op, env):
    tag = op[0]
    if tag == "enc":
        env[op[1]] = _pt(op[2])
    elif tag == "ew":
        kind, out, a, b = op[1], op[2], op[3], op[4]
        x = env[a]
        y = env[b] if kind.endswith("_ct") else _pt(b)
        if kind.startswith("add"):
            env[out] = (x + y) % Q
        elif kind.startswith("sub"):
            env[out] = (x - y) % Q
        else:
            env[out] = (x * y) % Q
    elif tag == "rot":
        env[op[1]] = np.roll(env[op[2]], -(op[3] % SLOTS))
    else:
        env[op[1]] = env[op[2]].copy()


def interpret(ops, plan=None, rank=0, allreduce=None):
    env = {}
    for i, op in enumerate(ops):
        if plan is not None:
            k = plan.kind[i]
            for vid in plan.reduce_before.get(i, ()):
                have = plan.present(plan.deps[vid], rank)
                env[vid] = allreduce(env[vid] if have else np.zeros(SLOTS, dtype=np.int64))
            if k == "join":
                a, b = plan.join_args[i]
                ha, hb = (plan.present(plan.deps[v], rank) for v in (a, b))
                if not (ha and hb):
                    if ha or hb:
                        env[op[2]] = env[a if ha else b]
                    continue
            elif isinstance(k, tuple) and k[1] != rank:
                continue
        _apply(op, env)
    return env


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, golden_dir, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19693_b200.dp import ShardPlan

    prog = _program(golden_dir, "c1_trace.npz")
    plan = ShardPlan(prog.ops, prog.n_setup, 3, world)

    def allreduce(v):
        t = torch.from_numpy(v.copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy() % Q

    env = interpret(prog.ops, plan, rank, allreduce)
    out[rank] = [env[o].tolist() for o in prog.outputs]
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_sharded_step_matches_sequential(golden_dir):
    prog = _program(golden_dir, "c1_trace.npz")
    seq = interpret(prog.ops)
    want = [seq[o].tolist() for o in prog.outputs]
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), golden_dir, out), nprocs=world, join=True)
    for rank in range(world):
        assert out[rank] == want
