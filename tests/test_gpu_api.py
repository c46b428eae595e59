"""HE-API semantics on the B200 backend, after the reference's backend tests
(/root/reference/pkg/tests/test_ckks_backend.py:25-174): zero / constant /
ragged encodings, the rotation group law, cross-level alignment, the debug
refresh with injected error, depth accounting identical to exact float
semantics on a random program, and empty-batch / zero-row C-ABI calls."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_19693_b200 import he_api  # noqa: E402
from paper_2506_19693_b200.scheme import make_params  # noqa: E402


@pytest.fixture(scope="module")
def small():
    params = make_params(level=10, scale_bits=40, poly_degree=2**12)
    return params, he_api.keygen(params, {1, 2, 3}, backend="ckks", rng_seed=4)


def _pl(params, v):
    return he_api.make_plain(v, params.slot_count, float(params.scale_bits))


def test_zero_constant_and_ragged_plaintexts(small):
    params, cust = small
    n = params.slot_count
    for v in (np.zeros(n), np.full(n, 0.75), np.array([0.5, -0.25, 1.0])):
        got = cust.decrypt(cust.encrypt(_pl(params, v))).values
        want = np.zeros(n)
        want[: v.shape[0]] = v  # a short vector fills the leading slots
        assert np.max(np.abs(got - want)) <= 2.0**-25


def test_rotation_group_law(small):
    params, cust = small
    ev = cust.evaluator
    v = np.random.default_rng(5).uniform(-1, 1, params.slot_count)
    ct = cust.encrypt(_pl(params, v))
    two_steps = cust.decrypt(ev.rotate(ev.rotate(ct, 1), 2)).values
    one_step = cust.decrypt(ev.rotate(ct, 3)).values
    assert np.max(np.abs(two_steps - one_step)) <= 2.0**-24
    assert np.max(np.abs(one_step - np.roll(v, -3))) <= 2.0**-24


def test_cross_level_alignment(small):
    params, cust = small
    ev = cust.evaluator
    rng = np.random.default_rng(6)
    v, w = rng.uniform(-1, 1, params.slot_count), rng.uniform(-1, 1, params.slot_count)
    cv, cw = cust.encrypt(_pl(params, v)), cust.encrypt(_pl(params, w))
    deep = ev.mul(ev.mul(cv, cw), cw)
    mixed = ev.add(deep, cv)
    assert mixed.level_remaining == deep.level_remaining
    assert np.max(np.abs(cust.decrypt(mixed).values - (v * w * w + v))) <= 2.0**-24


def test_debug_refresh_with_injected_error():
    params = make_params(level=3, scale_bits=40, poly_degree=2**10)
    cust = he_api.keygen(params, set(), backend="ckks", rng_seed=1, bootstrap_eps=2.0**-20)
    v = np.random.default_rng(0).uniform(-1, 1, params.slot_count)
    ct = cust.encrypt(_pl(params, v))
    before = cust.decrypt(ct).values
    refreshed = cust.bootstrap(ct)
    assert refreshed.level_remaining == params.refresh_level
    dev = np.max(np.abs(cust.decrypt(refreshed).values - before))
    assert 0.0 < dev <= 2.0**-19


def test_depth_accounting_matches_exact_semantics():
    """Values may differ from exact arithmetic by noise, depth and level
    accounting never: the same program on the B200 backend and on the exact
    float stand-in backend (tests/test_host.py) must agree."""
    from test_host import _FloatBackend  # tests/ is on sys.path under pytest

    params = make_params(level=6, scale_bits=40, poly_degree=2**10)
    n = params.slot_count
    gpu = he_api.keygen(params, {1, 2}, backend="ckks", rng_seed=2)
    cls = type("FB", (_FloatBackend, he_api.Backend), {})
    ref = he_api.KeyCustodian(cls(params, "exact"), {1, 2})

    def program(cust):
        ev = cust.evaluator
        r = np.random.default_rng(7)
        a = cust.encrypt(he_api.make_plain(r.uniform(-1, 1, n), n, 40.0))
        b = cust.encrypt(he_api.make_plain(r.uniform(-1, 1, n), n, 40.0))
        with cust.ledger.iteration():
            t = ev.mul(a, b)
            t = ev.add(t, ev.rotate(a, 1))
            t = ev.mul(t, t)
            t = ev.sub(t, b)
            t = ev.mul(t, he_api.make_plain(np.full(n, 0.5), n, 40.0))
        return cust.ledger.iteration_depths[-1], t

    (d_gpu, t_gpu), (d_ref, t_ref) = program(gpu), program(ref)
    assert d_gpu == d_ref == 3
    assert (t_gpu.level_remaining, t_gpu.depth) == (t_ref.level_remaining, t_ref.depth)
    err = np.max(np.abs(gpu.decrypt(t_gpu).values - ref.decrypt(t_ref).values))
    assert err <= 2.0**-20


def test_empty_batches_are_no_ops(small):
    """Zero rows / zero items through the C-ABI: status 0, nothing touched."""
    from paper_2506_19693_b200 import _native as nat

    params, cust = small
    ch = cust.backend.chain
    buf = torch.zeros(1, dtype=torch.uint64, device="cuda")
    lm = ch.q_map(1)
    assert nat.LIB.ckb_ntt_forward(ch.ring_p, nat.ptr(buf), 0, 1, lm, nat.stream_handle()) == 0
    assert nat.LIB.ckb_elementwise(ch.ring_p, 0, nat.ptr(buf), nat.ptr(buf), nat.ptr(buf), None,
                                   0, 1, lm, 0, nat.stream_handle()) == 0
    torch.cuda.synchronize()
    assert int(buf.view(torch.int64)[0]) == 0


def test_streaming_pipeline_matches_direct(small):
    """streaming.Pipeline (chunked H2D / compute / D2H on three streams) gives
    the same planes as one direct batched call."""
    from paper_2506_19693_b200.streaming import Pipeline

    params, cust = small
    be = cust.backend
    lvl = params.level
    m = be.chain.level_limbs[lvl]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)

    def rand_batch(b):
        t = torch.empty(b, 2, m, be.n, dtype=torch.int64, device="cuda")
        for i, p in enumerate(be.chain.limbs_at(lvl)):
            t[:, :, i].random_(0, p, generator=gen)
        return t.view(torch.uint64)

    a, b = rand_batch(5), rand_batch(5)
    steps = [1, 2, 3, 1, 2]
    want_m = be.batch_hmult(a, b, lvl).cpu()
    want_r = be.batch_hrot(a, steps, lvl).cpu()
    ha, hb = a.cpu().pin_memory(), b.cpu().pin_memory()
    om = torch.empty_like(want_m).pin_memory()
    orr = torch.empty_like(want_r).pin_memory()
    Pipeline().run(lambda d, lo, hi: [be.batch_hmult(d[0], d[1], lvl),
                                      be.batch_hrot(d[0], steps[lo:hi], lvl)],
                   [ha, hb], [om, orr], chunk=2)
    torch.cuda.synchronize()
    assert torch.equal(om.view(torch.int64), want_m.view(torch.int64))
    assert torch.equal(orr.view(torch.int64), want_r.view(torch.int64))
