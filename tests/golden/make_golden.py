"""Generate the golden fixtures from the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--c1-ckks]

Outputs (committed):
  ref_ntt.npz        NttPlan forward/inverse vectors      (ckks/ntt.py:100-154)
  ref_ckks_n512.npz  CkksBackend ciphertext planes for encrypt/add/sub/mul_ct/
                     mul_pt/add_pt/rotate/cross-level add (ckks/backend.py), the
                     secret, the prime chain and SHA-256 digests of every key row
  ref_rbot_n512.npz  a reference RBOT model container (serialize.py) of a
                     2-block model with its RBKY key file and decrypted payloads
  c1_trace.npz       the HE-API call sequence of one unchanged
                     nn.train_iteration (config 1 shape: 16->8->2, batch 32,
                     N=2^12, L=8) recorded on the sim backend, plus the sim
                     backend's decrypted weights after the step; with
                     --c1-ckks also the reference CkksBackend's weights (~3 min).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def ct_planes(cv):
    ct = cv.payload
    return np.stack([ct.c0.to_coeff().planes.astype(np.uint64),
                     ct.c1.to_coeff().planes.astype(np.uint64)])


def key_digest(ksk) -> str:
    h = hashlib.sha256()
    for b, a in zip(ksk.rows_b, ksk.rows_a):
        h.update(np.ascontiguousarray(b.planes.astype("<u8")).tobytes())
        h.update(np.ascontiguousarray(a.planes.astype("<u8")).tobytes())
    return h.hexdigest()


def make_ntt():
    from ciphermlp.ckks.ntt import NttPlan, nearest_ntt_prime

    out = {}
    rng = np.random.default_rng(2024)
    for n, target in ((16, 1 << 27), (64, 1 << 27), (1024, 1 << 30), (4096, 1 << 30),
                      (8192, 1 << 29)):
        p = nearest_ntt_prime(target, 2 * n, set())
        plan = NttPlan(p, n)
        a = rng.integers(0, p, n, dtype=np.uint64)
        out[f"n{n}_p"] = np.array([p], dtype=np.uint64)
        out[f"n{n}_in"] = a
        out[f"n{n}_fwd"] = plan.forward(a)
        out[f"n{n}_inv"] = plan.inverse(a)
        out[f"n{n}_psi_brv"] = plan.psi_brv[: min(n, 64)]
    np.savez_compressed(os.path.join(HERE, "ref_ntt.npz"), **out)


def make_ckks():
    from ciphermlp.api import keygen, make_plain
    from ciphermlp.params import make_params

    n = 512
    params = make_params(level=3, scale_bits=40, poly_degree=n)
    rots = {1, 3, -1}
    cust = keygen(params, rots, backend="ckks", rng_seed=11)
    be = cust.backend
    ev = cust.evaluator
    slots = params.slot_count
    rng = np.random.default_rng(5)
    v1, v2, v3 = (rng.uniform(-1, 1, slots) for _ in range(3))
    pl = lambda v: make_plain(v, slots, 40.0)
    ct1 = cust.encrypt(pl(v1))
    ct2 = cust.encrypt(pl(v2))
    out = {
        "params": np.array([n, 3, 40], dtype=np.int64),
        "chain": np.array(params.modulus_chain, dtype=np.int64),
        "rots": np.array(sorted(rots), dtype=np.int64),
        "rng_seed": np.array([11], dtype=np.int64),
        "all_primes": np.array(be.ctx.all_primes, dtype=np.uint64),
        "level_limbs": np.array(be.ctx.level_limbs, dtype=np.int64),
        "scale_at": np.array(be.ctx.scale_at, dtype=np.float64),
        "secret": be.sk.coeffs.astype(np.int8),
        "v1": v1, "v2": v2, "v3": v3,
        "ct1": ct_planes(ct1), "ct2": ct_planes(ct2),
        "ct1_serial": np.array([ct1.serial], dtype=np.int64),
        "ct2_serial": np.array([ct2.serial], dtype=np.int64),
    }
    digests = {"relin": key_digest(be.eval_keys.relin)}
    for g, k in sorted(be.eval_keys.rotations.items()):
        digests[f"rot_{g}"] = key_digest(k)
    out["key_digests"] = np.array(json.dumps(digests))
    ops = {
        "add": ev.add(ct1, ct2),
        "sub": ev.sub(ct1, ct2),
        "mul": ev.mul(ct1, ct2),
        "rot1": ev.rotate(ct1, 1),
        "rot3": ev.rotate(ct1, 3),
        "rotm1": ev.rotate(ct1, -1),
    }
    # plaintext operands: record the exact integer encoding the reference used
    lvl = ct1.level_remaining
    out["pt3_coeffs"] = be.encoder.embed(v3, be.ctx.scale_at[lvl]).astype(np.int64)
    out["pt3neg_coeffs"] = be.encoder.embed(-v3, be.ctx.scale_at[lvl]).astype(np.int64)
    ops["mul_pt"] = ev.mul(ct1, pl(v3))
    ops["add_pt"] = ev.add(ct1, pl(v3))
    ops["sub_pt"] = ev.sub(ct1, pl(v3))
    deep = ev.mul(ev.mul(ct1, ct2), ct2)
    ops["deep"] = deep
    ops["mixed"] = ev.add(deep, ct1)
    ops["sq"] = ev.mul(ops["mul"], ops["mul"])
    for name, cv in ops.items():
        out[f"out_{name}"] = ct_planes(cv)
        out[f"lvl_{name}"] = np.array([cv.level_remaining], dtype=np.int64)
        out[f"dec_{name}"] = cust.decrypt(cv).values
    out["dec_ct1"] = cust.decrypt(ct1).values
    # the reference's own serialisations (RBCT ciphertext, RBKY key container)
    from ciphermlp.ckks.backend import save_custodian

    out["rbct_ct1"] = np.frombuffer(be.serialize_cipher(ct1), dtype=np.uint8)
    out["rbct_mul"] = np.frombuffer(be.serialize_cipher(ops["mul"]), dtype=np.uint8)
    out["rbky"] = np.frombuffer(save_custodian(cust), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "ref_ckks_n512.npz"), **out)


# ---------------------------------------------------------------------------
# config-1 training trace
# ---------------------------------------------------------------------------


def c1_setup():
    """Config 1 (BASELINE.json configs[0]) shaped synthetic run."""
    from ciphermlp.packing import Architecture, compute_dims

    arch = Architecture(16, (8,), 2)
    n = 2**12
    rng = np.random.default_rng(20250624)
    x = rng.uniform(-1, 1, size=(32, 16))
    teacher = rng.normal(size=(16, 2))
    y = np.argmax(x @ teacher, axis=1)
    onehot = np.eye(2)[y]
    # Xavier-uniform init (BASELINE config 1), overriding nn.init_weights
    w1 = rng.uniform(-1, 1, size=(16, 8)) * np.sqrt(6.0 / (16 + 8))
    c1 = rng.uniform(-1, 1, size=(8, 2)) * np.sqrt(6.0 / (8 + 2))
    shape = compute_dims(arch, n // 2)
    return arch, n, x, onehot, w1, c1, shape


def build_c1(backend: str, **opts):
    from ciphermlp.api import keygen
    from ciphermlp.nn import Hyperparams, build_model, layer_format, classifier_format
    from ciphermlp.packing import encrypt_packed, pack, required_rotations
    from ciphermlp.params import make_params
    from ciphermlp.depth import tau_total

    arch, n, x, onehot, w1, c1, shape = c1_setup()
    params = make_params(level=tau_total(1), scale_bits=40, poly_degree=n)
    cust = keygen(params, required_rotations(shape), backend=backend, **opts)
    hyper = Hyperparams(learning_rate=0.05, momentum=0.9, iterations=1, batch_size=32, rng_seed=0)
    model = build_model(arch, params, hyper, cust)
    blk = model.blocks[0]
    blk.layer_weights = encrypt_packed(cust, pack(w1, layer_format(blk.kind), shape))
    blk.classifier_weights = encrypt_packed(cust, pack(c1, classifier_format(blk.kind), shape))
    return cust, model, shape, x, onehot


def run_c1(cust, model, shape, x, onehot):
    from ciphermlp.nn import prepare_sample, train_iteration

    batch = [prepare_sample(x[i], onehot[i], shape, cust) for i in range(x.shape[0])]
    train_iteration(model, batch, cust, 1)
    return model


def weights_of(model, cust):
    b = model.blocks[0]
    return np.stack([cust.decrypt(pm.payload).values
                     for pm in (b.layer_weights, b.classifier_weights,
                                b.layer_velocity, b.classifier_velocity)])


def make_c1_trace(with_ckks: bool):
    from ciphermlp.api import CipherVector, PlainVector
    from ciphermlp.simbackend import SimBackend

    ops: list = []
    pts: dict = {}
    ids: dict = {}

    def pt_id(pv):
        key = pv.values.tobytes()
        if key not in pts:
            pts[key] = len(pts)
        return pts[key]

    def cid(cv):
        return ids[cv.serial]

    def new(cv):
        ids[cv.serial] = len(ids)
        return ids[cv.serial]

    class Recording(SimBackend):
        def encrypt(self, pv):
            cv = super().encrypt(pv)
            ops.append(["enc", new(cv), pt_id(pv)])
            return cv

        def elementwise(self, kind, a, b):
            cv = super().elementwise(kind, a, b)
            arg = cid(b) if isinstance(b, CipherVector) else pt_id(b)
            ops.append(["ew", kind, new(cv), cid(a), arg])
            return cv

        def rotate(self, a, k, allowed):
            cv = super().rotate(a, k, allowed)
            ops.append(["rot", new(cv), cid(a), int(k)])
            return cv

        def bootstrap(self, cv):
            out = super().bootstrap(cv)
            ops.append(["bs", new(out), cid(cv)])
            return out

    import ciphermlp.simbackend as sb

    orig = sb.SimBackend
    sb.SimBackend = Recording
    try:
        cust, model, shape, x, onehot = build_c1("sim")
        n_setup = len(ops)
        run_c1(cust, model, shape, x, onehot)
    finally:
        sb.SimBackend = orig
    b = model.blocks[0]
    outs = [cid(pm.payload) for pm in (b.layer_weights, b.classifier_weights,
                                       b.layer_velocity, b.classifier_velocity)]
    sim_w = weights_of(model, cust)
    pt_arr = np.zeros((len(pts), shape.slots))
    for k, i in pts.items():
        pt_arr[i] = np.frombuffer(k, dtype=np.float64)
    from ciphermlp.packing import required_rotations

    res = {
        "ops": np.array(json.dumps(ops)),
        "n_setup": np.array([n_setup]),
        "plaintexts": pt_arr,
        "outputs": np.array(outs),
        "rotations": np.array(sorted(required_rotations(shape))),
        "params": np.array([2**12, 8, 40]),
        "sim_weights": sim_w,
    }
    if with_ckks:
        import time

        t0 = time.perf_counter()
        cust, model, shape, x, onehot = build_c1("ckks", rng_seed=3)
        t1 = time.perf_counter()
        run_c1(cust, model, shape, x, onehot)
        t2 = time.perf_counter()
        res["ckks_weights"] = weights_of(model, cust)
        res["ckks_seconds"] = np.array([t1 - t0, t2 - t1])
        print(f"reference CKKS: setup {t1 - t0:.1f}s, train_iteration {t2 - t1:.1f}s")
    np.savez_compressed(os.path.join(HERE, "c1_trace.npz"), **res)
    kinds = {}
    for op in ops:
        key = op[1] if op[0] == "ew" else op[0]
        kinds[key] = kinds.get(key, 0) + 1
    print("c1 trace ops:", kinds, "plaintexts:", len(pts))


def make_c4_trace(lr: float = 0.005):
    """Config 4 with the survey's substitution: 196-feature
    14x14 inputs (pixels U[0,1]), 196->128->10, 10 uniform random classes,
    batch 128, N=2^16, L = tau(1) + 16 = 24 with bootstrap_depth 16, Xavier
    init; one train_iteration recorded on the sim backend (the refresh calls
    become real bootstrapping on the B200)."""
    from ciphermlp.api import CipherVector, keygen
    from ciphermlp.depth import tau_total
    from ciphermlp.nn import (Hyperparams, build_model, classifier_format, layer_format,
                              prepare_sample, train_iteration)
    from ciphermlp.packing import Architecture, compute_dims, encrypt_packed, pack, required_rotations
    from ciphermlp.params import make_params
    import ciphermlp.simbackend as sb

    arch = Architecture(196, (128,), 10)
    n = 2**16
    params = make_params(level=tau_total(1) + 16, scale_bits=45, poly_degree=n,
                         bootstrap_depth=16)
    shape = compute_dims(arch, n // 2)
    rng = np.random.default_rng(20250704)
    bsz = 128
    x = rng.uniform(0, 1, size=(bsz, 196))
    y = rng.integers(0, 10, bsz)
    onehot = np.eye(10)[y]
    w1 = rng.uniform(-1, 1, size=(196, 128)) * np.sqrt(6.0 / (196 + 128))
    c1 = rng.uniform(-1, 1, size=(128, 10)) * np.sqrt(6.0 / (128 + 10))

    ops, pts, ids = [], {}, {}

    def pt_id(pv):
        key = pv.values.tobytes()
        if key not in pts:
            pts[key] = len(pts)
        return pts[key]

    class Recording(sb.SimBackend):
        def encrypt(self, pv):
            cv = super().encrypt(pv)
            ids[cv.serial] = len(ids)
            ops.append(["enc", ids[cv.serial], pt_id(pv)])
            return cv

        def elementwise(self, kind, a, b):
            cv = super().elementwise(kind, a, b)
            arg = ids[b.serial] if isinstance(b, CipherVector) else pt_id(b)
            ids[cv.serial] = len(ids)
            ops.append(["ew", kind, ids[cv.serial], ids[a.serial], arg])
            return cv

        def rotate(self, a, k, allowed):
            cv = super().rotate(a, k, allowed)
            ids[cv.serial] = len(ids)
            ops.append(["rot", ids[cv.serial], ids[a.serial], int(k)])
            return cv

        def bootstrap(self, cv):
            out = super().bootstrap(cv)
            ids[out.serial] = len(ids)
            ops.append(["bs", ids[out.serial], ids[cv.serial]])
            return out

    orig = sb.SimBackend
    sb.SimBackend = Recording
    try:
        cust = keygen(params, required_rotations(shape), backend="sim")
        # lr 0.005 (as config 5): with 0.05 the exact model's second step already
        # diverges (classifier velocity ~5e6), far outside what CKKS can carry
        hyper = Hyperparams(learning_rate=lr, momentum=0.9, iterations=1, batch_size=bsz)
        model = build_model(arch, params, hyper, cust)
        blk = model.blocks[0]
        blk.layer_weights = encrypt_packed(cust, pack(w1, layer_format(blk.kind), shape))
        blk.classifier_weights = encrypt_packed(cust, pack(c1, classifier_format(blk.kind), shape))
        n_setup = len(ops)
        batch = [prepare_sample(x[i], onehot[i], shape, cust) for i in range(bsz)]
        train_iteration(model, batch, cust, 1)
        b = model.blocks[0]
        state = (b.layer_weights, b.classifier_weights, b.layer_velocity, b.classifier_velocity)
        outs = [ids[pm.payload.serial] for pm in state]
        sim_w = np.stack([cust.decrypt(pm.payload).values for pm in state])
        # step 2 (steady state: the refreshed weights and velocities sit at the
        # refresh level) on the next minibatch of the same generator
        s2 = len(ops)
        x2 = rng.uniform(0, 1, size=(bsz, 196))
        onehot2 = np.eye(10)[rng.integers(0, 10, bsz)]
        batch2 = [prepare_sample(x2[i], onehot2[i], shape, cust) for i in range(bsz)]
        train_iteration(model, batch2, cust, 2)
        state = (b.layer_weights, b.classifier_weights, b.layer_velocity, b.classifier_velocity)
        outs2 = [ids[pm.payload.serial] for pm in state]
        sim_w2 = np.stack([cust.decrypt(pm.payload).values for pm in state])
    finally:
        sb.SimBackend = orig
    ops2 = ops[s2:]
    ops = ops[:s2]
    pt_arr = np.zeros((len(pts), shape.slots))
    for k, i in pts.items():
        pt_arr[i] = np.frombuffer(k, dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "c4_trace.npz"), ops=np.array(json.dumps(ops)),
                        n_setup=np.array([n_setup]), plaintexts=pt_arr, outputs=np.array(outs),
                        rotations=np.array(sorted(required_rotations(shape))),
                        params=np.array([n, params.level, 45, 16]), sim_weights=sim_w,
                        grid=np.array([shape.r, shape.c]), ops_step2=np.array(json.dumps(ops2)),
                        outputs_step2=np.array(outs2), sim_weights_step2=sim_w2)
    kinds = {}
    for op in ops:
        key = op[1] if op[0] == "ew" else op[0]
        kinds[key] = kinds.get(key, 0) + 1
    print("c4 trace ops:", kinds, "plaintexts:", len(pts), "grid", shape)


def make_c5_trace(init_scale: float = 0.25, lr: float = 0.005, out: str = "c5_trace.npz"):
    """Config 5 (deep tabular): 64 N(0,1) features, binary labels from a seeded
    random two-layer teacher, 64->64->64->64->64->2 local-error-signal MLP,
    batch 256, N=2^16, L = tau(4) + 16 = 32 with bootstrap_depth 16 (above the
    128-bit bound: insecure-test), Xavier init; one
    train_iteration recorded on the sim backend like config 4."""
    from ciphermlp.api import CipherVector, keygen
    from ciphermlp.depth import tau_total
    from ciphermlp.nn import (Hyperparams, build_model, classifier_format, layer_format,
                              prepare_sample, train_iteration)
    from ciphermlp.packing import Architecture, compute_dims, encrypt_packed, pack, required_rotations
    from ciphermlp.params import make_params
    import ciphermlp.simbackend as sb

    hidden = (64, 64, 64, 64)
    arch = Architecture(64, hidden, 2)
    n = 2**16
    params = make_params(level=tau_total(len(hidden)) + 16, scale_bits=45, poly_degree=n,
                         bootstrap_depth=16)  # security_claim defaults to insecure-test
    shape = compute_dims(arch, n // 2)
    rng = np.random.default_rng(20250705)
    bsz = 256
    x = rng.normal(0, 1, size=(bsz, 64))
    t1 = rng.normal(0, 1, size=(64, 16))
    t2 = rng.normal(0, 1, size=(16, 2))
    y = np.argmax(np.tanh(x @ t1) @ t2, axis=1)
    onehot = np.eye(2)[y]

    ops, pts, ids = [], {}, {}

    def pt_id(pv):
        key = pv.values.tobytes()
        if key not in pts:
            pts[key] = len(pts)
        return pts[key]

    class Recording(sb.SimBackend):
        def encrypt(self, pv):
            cv = super().encrypt(pv)
            ids[cv.serial] = len(ids)
            ops.append(["enc", ids[cv.serial], pt_id(pv)])
            return cv

        def elementwise(self, kind, a, b):
            cv = super().elementwise(kind, a, b)
            arg = ids[b.serial] if isinstance(b, CipherVector) else pt_id(b)
            ids[cv.serial] = len(ids)
            ops.append(["ew", kind, ids[cv.serial], ids[a.serial], arg])
            return cv

        def rotate(self, a, k, allowed):
            cv = super().rotate(a, k, allowed)
            ids[cv.serial] = len(ids)
            ops.append(["rot", ids[cv.serial], ids[a.serial], int(k)])
            return cv

        def bootstrap(self, cv):
            out = super().bootstrap(cv)
            ids[out.serial] = len(ids)
            ops.append(["bs", ids[out.serial], ids[cv.serial]])
            return out

    orig = sb.SimBackend
    sb.SimBackend = Recording
    try:
        cust = keygen(params, required_rotations(shape), backend="sim")
        hyper = Hyperparams(learning_rate=lr, momentum=0.9, iterations=1, batch_size=bsz)
        model = build_model(arch, params, hyper, cust)
        dims = (64,) + hidden
        for k, blk in enumerate(model.blocks):
            fan_in, fan_out = dims[k], hidden[k]
            w = rng.uniform(-1, 1, size=(fan_in, fan_out)) * np.sqrt(6.0 / (fan_in + fan_out))
            c = rng.uniform(-1, 1, size=(fan_out, 2)) * np.sqrt(6.0 / (fan_out + 2))
            w, c = w * init_scale, c * init_scale  # keeps the depth-4 z^2+z stack bounded
            blk.layer_weights = encrypt_packed(cust, pack(w, layer_format(blk.kind), shape))
            blk.classifier_weights = encrypt_packed(cust, pack(c, classifier_format(blk.kind),
                                                               shape))
        n_setup = len(ops)
        batch = [prepare_sample(x[i], onehot[i], shape, cust) for i in range(bsz)]
        train_iteration(model, batch, cust, 1)

        def state():
            o, w = [], []
            for b in model.blocks:
                for pm in (b.layer_weights, b.classifier_weights, b.layer_velocity,
                           b.classifier_velocity):
                    o.append(ids[pm.payload.serial])
                    w.append(cust.decrypt(pm.payload).values)
            return o, w

        outs, sim_w = state()
        # step 2 (steady state, refreshed weights) on the next minibatch
        s2 = len(ops)
        x2 = rng.normal(0, 1, size=(bsz, 64))
        onehot2 = np.eye(2)[np.argmax(np.tanh(x2 @ t1) @ t2, axis=1)]
        batch2 = [prepare_sample(x2[i], onehot2[i], shape, cust) for i in range(bsz)]
        train_iteration(model, batch2, cust, 2)
        outs2, sim_w2 = state()
    finally:
        sb.SimBackend = orig
    ops2 = ops[s2:]
    ops = ops[:s2]
    pt_arr = np.zeros((len(pts), shape.slots))
    for k, i in pts.items():
        pt_arr[i] = np.frombuffer(k, dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, out), ops=np.array(json.dumps(ops)),
                        n_setup=np.array([n_setup]), plaintexts=pt_arr, outputs=np.array(outs),
                        rotations=np.array(sorted(required_rotations(shape))),
                        params=np.array([n, params.level, 45, 16]), sim_weights=np.stack(sim_w),
                        grid=np.array([shape.r, shape.c]), ops_step2=np.array(json.dumps(ops2)),
                        outputs_step2=np.array(outs2), sim_weights_step2=np.stack(sim_w2))
    kinds = {}
    for op in ops:
        key = op[1] if op[0] == "ew" else op[0]
        kinds[key] = kinds.get(key, 0) + 1
    print("c5 trace ops:", kinds, "plaintexts:", len(pts), "grid", shape,
          "max |weights, velocities| per block:",
          [round(float(np.abs(v).max()), 3) for v in sim_w])


def make_rbot():
    """RBOT model container (serialize.py:38-60) of a freshly built 4->4->4->2
    model (one RE and one CE block) under the n512 keyset, with its RBKY key
    file and the decrypted values of all 8 payloads."""
    from ciphermlp.api import keygen
    from ciphermlp.ckks.backend import save_custodian
    from ciphermlp.nn import Hyperparams, build_model
    from ciphermlp.packing import Architecture
    from ciphermlp.params import make_params
    from ciphermlp.serialize import save_model

    n = 512
    params = make_params(level=3, scale_bits=40, poly_degree=n)
    cust = keygen(params, {1, 3, -1}, backend="ckks", rng_seed=11)
    arch = Architecture(4, (4, 4), 2)
    model = build_model(arch, params, Hyperparams(learning_rate=0.05, rng_seed=3), cust)
    out = {"rbky": np.frombuffer(save_custodian(cust), dtype=np.uint8),
           "rbot": np.frombuffer(save_model(model, cust), dtype=np.uint8)}
    dec = []
    for b in model.blocks:
        for pm in (b.layer_weights, b.classifier_weights, b.layer_velocity,
                   b.classifier_velocity):
            dec.append(cust.decrypt(pm.payload).values)
    out["dec"] = np.stack(dec)
    np.savez_compressed(os.path.join(HERE, "ref_rbot_n512.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1-ckks", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    if a.only in ("", "ntt"):
        make_ntt()
    if a.only in ("", "ckks"):
        make_ckks()
    if a.only in ("", "rbot"):
        make_rbot()
    if a.only in ("", "c1"):
        make_c1_trace(a.c1_ckks)
    if a.only == "c4":
        make_c4_trace()
    if a.only == "c5":
        make_c5_trace()


if __name__ == "__main__":
    sys.exit(main())
