"""WaveExecutor planning on the recorded traces (host logic, CPU): dependency
waves and the rotate-and-accumulate fusion (executor._plan_fusion)."""

import os
import types

import pytest

from paper_2506_19693_b200.executor import WaveExecutor, _inputs
from paper_2506_19693_b200.replay import Program


def _stub_custodian(prog, real_bootstrap=False):
    params = types.SimpleNamespace(level=30, refresh_level=8, slot_count=1 << 15)
    be = types.SimpleNamespace(params=params, real_bootstrap=real_bootstrap)
    return types.SimpleNamespace(backend=be)


@pytest.mark.parametrize("name,n_rot", [("c1_trace.npz", 704), ("c4_trace.npz", 3840),
                                        ("c5_trace.npz", 32256)])
def test_every_rotation_fuses_with_its_accumulate(golden_dir, name, n_rot):
    prog = Program.load(os.path.join(golden_dir, name))
    ex = WaveExecutor(prog, _stub_custodian(prog, real_bootstrap=name != "c1_trace.npz"))
    ops = prog.ops
    assert sum(op[0] == "rot" for op in ops[prog.n_setup:]) == n_rot
    assert len(ex.fuse) == n_rot and len(ex.fused_adds) == n_rot
    readers = {}
    for k, op in enumerate(ops):
        for x in _inputs(op):
            readers.setdefault(x, []).append(k)
    wave_of = {x: w for w, wave in enumerate(ex.waves) for x in wave}
    outputs = set(prog.outputs)
    for i, j in ex.fuse.items():
        rot, add = ops[i], ops[j]
        assert rot[0] == "rot" and add[0] == "ew" and add[1] == "add_ct"
        assert {add[3], add[4]} == {rot[1], rot[2]}
        # the rotation's output has no other reader and is not a program output
        assert readers[rot[1]] == [j] and rot[1] not in outputs
        # the add runs in a later wave than the rotation (it is skipped there)
        assert wave_of[j] > wave_of[i]


def test_fusion_skips_rotations_with_other_readers(golden_dir):
    prog = Program.load(os.path.join(golden_dir, "c1_trace.npz"))
    i = next(k for k, op in enumerate(prog.ops) if op[0] == "rot" and k >= prog.n_setup)
    out = prog.ops[i][1]
    # make the rotation's output a program output: it must then be materialised
    prog.outputs = list(prog.outputs) + [out]
    ex = WaveExecutor(prog, _stub_custodian(prog))
    assert i not in ex.fuse


@pytest.mark.parametrize("name,n_bs", [("c4_trace.npz", 4), ("c5_trace.npz", 16)])
def test_steady_step_program(golden_dir, name, n_bs):
    """The recorded second train_iteration: step 1 keeps exactly the state it
    reads (its refreshed weights and velocities), step 2 starts after step 1,
    reads nothing else from it, and its real bootstraps are deferred into one
    batched final wave."""
    path = os.path.join(golden_dir, name)
    p1 = Program.load(path)
    p2 = Program.load_step2(path)
    assert p1.carry == set(p1.outputs)
    assert p2.n_setup == len(p1.ops) and p2.ops[: len(p1.ops)] == p1.ops
    defined_before = {op[2] if op[0] == "ew" else op[1] for op in p1.ops}
    reads = {x for op in p2.ops[p2.n_setup:] for x in _inputs(op)}
    defined_after = {op[2] if op[0] == "ew" else op[1] for op in p2.ops[p2.n_setup:]}
    assert (reads - defined_after) <= p1.keep and not (defined_after & defined_before)
    ex = WaveExecutor(p2, _stub_custodian(p2, real_bootstrap=True))
    bs = [i for i, op in enumerate(p2.ops) if op[0] == "bs" and i >= p2.n_setup]
    assert len(bs) == n_bs and sorted(ex.waves[-1]) == bs
    # step-2 levels start from the refresh level: every op after setup sits at
    # or below it (the step consumes user levels only)
    assert max(ex.level_of[op[2] if op[0] == "ew" else op[1]]
               for op in p2.ops[p2.n_setup:] if op[0] != "enc") <= 8


@pytest.mark.parametrize("name,n_sums,leaves,waves_max", [
    ("c1_trace.npz", 2, 32, 70), ("c4_trace.npz", 2, 128, 80), ("c5_trace.npz", 8, 256, 160)])
def test_fold_chains_become_summation_trees(golden_dir, name, n_sums, leaves, waves_max):
    """executor._plan_sums: the delta-W fold (nn.py:373-381, acc = acc + dW_s
    over the batch) becomes one n-ary sum per block and weight kind; the inner
    adds leave the wave plan, every leaf is read by the sum, the values a sum
    replaces have no other reader, and the step's waves shrink accordingly."""
    prog = Program.load(os.path.join(golden_dir, name))
    ex = WaveExecutor(prog, _stub_custodian(prog, real_bootstrap=name != "c1_trace.npz"))
    assert len(ex.sums) == n_sums
    assert all(len(v) == leaves for v in ex.sums.values())
    assert len(ex.absorbed) == n_sums * (leaves - 2)
    planned = {i for wave in ex.waves for i in wave}
    assert not (planned & ex.absorbed) and set(ex.sums) <= planned
    readers = {}
    for k, op in enumerate(prog.ops):
        for x in _inputs(op):
            readers.setdefault(x, []).append(k)
    for j in ex.absorbed:  # an absorbed add's result feeds exactly one add of its tree
        out = prog.ops[j][2]
        assert len(readers[out]) == 1 and out not in prog.keep
    for root, lv in ex.sums.items():  # each leaf's last use is its sum
        assert all(ex.last_use[x] >= root for x in lv)
    assert len(ex.waves) <= waves_max


def test_data_parallel_executor_keeps_the_fold_joins():
    from paper_2506_19693_b200.dp import DataParallelExecutor

    assert DataParallelExecutor.rewrite_sums is False
