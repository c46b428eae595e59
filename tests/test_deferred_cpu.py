"""deferred.Recorder bookkeeping (host logic, CPU): operands, plaintext
de-duplication, output ids and recorded serials — what the first flush hands
to executor.WaveExecutor."""

import numpy as np

from paper_2506_19693_b200.deferred import LazyPayload, Recorder, _Program


class _Payload:
    def __init__(self, level):
        self.level = level


def test_recorder_builds_the_program_the_executor_reads():
    rec = Recorder(backend=None)
    x, y = _Payload(5), _Payload(5)
    v = np.linspace(-1, 1, 8)
    e1 = rec.record(("enc", None, rec.plaintext(v)), 7, serial=11)
    e2 = rec.record(("enc", None, rec.plaintext(v.copy())), 7, serial=13)
    s = rec.record(("ew", "add_ct", None, rec.operand(e1), rec.operand(e2)), 7)
    r = rec.record(("rot", None, rec.operand(s), 3), 7)
    m = rec.record(("ew", "mul_pt", None, rec.operand(x), rec.plaintext(-v)), 4)
    t = rec.record(("ew", "add_ct", None, rec.operand(y), rec.operand(x)), 5)
    assert all(isinstance(p, LazyPayload) for p in (e1, e2, s, r, m, t))
    assert len(rec.pt_rows) == 2  # equal plaintext vectors are encoded once
    assert rec.ops[0] == ("enc", e1.vid, 0) and rec.ops[1] == ("enc", e2.vid, 0)
    assert rec.ops[2] == ("ew", "add_ct", s.vid, e1.vid, e2.vid)
    assert rec.ops[3] == ("rot", r.vid, s.vid, 3)
    assert rec.serials == {0: 11, 1: 13}  # the eager hooks' RNG serials, by op index
    # a materialised operand is registered once, as a program input
    assert rec.ops[4][3] == rec.ops[5][4] and set(rec.inputs) == {rec.ops[4][3], rec.ops[5][3]}
    assert rec.inputs[rec.ops[4][3]] is x
    # outputs still referenced by the caller are what a flush keeps
    live = dict(rec.lazy)
    assert set(live) == {p.vid for p in (e1, e2, s, r, m, t)}
    prog = _Program(rec.ops, np.stack(rec.pt_rows), [v_ for v_ in live if v_ not in rec.inputs])
    assert prog._last_use[s.vid] == 3 and prog.keep == set(live)


def test_resolved_payloads_become_inputs_of_the_next_program():
    rec = Recorder(backend=None)
    lp = rec.new(3)
    done = _Payload(3)
    lp.value = done  # as after a flush
    vid = rec.operand(lp)
    assert rec.inputs[vid] is done and rec.operand(done) == vid


def test_pipelined_flushes_run_in_order_and_chain_pending_values():
    """deferred_async (pipelined): flush() returns at once; programs run in flush
    order on one worker; a value of a still-pending program enters the next
    program as an input and is read when that program runs; resolve() joins."""
    import threading
    import time

    class _Be:
        device = "cpu"

    rec = Recorder(backend=_Be(), pipelined=True)
    gate = threading.Event()
    ran = []

    def fake_run(snap, restore_serials):
        ops, serials, inputs, live, pts = snap
        assert restore_serials is False  # the recording thread owns the live counter
        gate.wait(5)
        for k, v in inputs.items():  # earlier programs have produced their values
            if isinstance(v, LazyPayload):
                assert v.value is not None
        ran.append([op[0] for op in ops])
        for vid, lp in live.items():
            lp.value = _Payload(lp.level)

    rec._run = fake_run
    issued = []
    a = rec.record(("enc", None, rec.plaintext(np.ones(4))), 5, serial=1)
    rec.flush(on_issued=lambda: issued.append(1))
    assert a.value is None and rec._pending  # returned before the program ran
    vid = rec.operand(a)  # pending value of program 1 -> input of program 2
    assert rec.inputs[vid] is a
    b = rec.record(("rot", None, vid, 1), 5)
    rec.flush(on_issued=lambda: issued.append(2))
    time.sleep(0.05)
    assert ran == []  # still gated
    gate.set()
    assert rec.resolve(b) is b.value  # joins every pending program
    assert ran == [["enc"], ["rot"]] and issued == [1, 2]
    assert a.value is not None and not rec._pending
