"""Benchmark: BASELINE.json config 2 (HE primitive sweep) on the B200 backend.

Workload (one "step"): a batch of 64 ciphertexts at N=2^16, L=24 40-bit limbs,
hybrid key switching dnum=3 with k=6 60-bit special primes:
  * NTT + iNTT of every limb of the batch,
  * ct x ct multiply + relinearise + rescale of 64 pairs (HMult),
  * rotation of 64 ciphertexts by 64 seeded steps in [1, 2^15), 64 keys (HRot).
Inputs are uniformly random limbs (seeded), resident in HBM (1.5 GiB per
operand batch, larger than the 126 MB L2, so no flush is needed).

metric  = BASELINE's "encrypted train ms/step; bootstrap ms; keyswitch GB/s vs
          HBM peak"; value = key-switching throughput: algorithmic bytes of the
          HMult + HRot batches (BASELINE.md §3 formulas, each distinct key once
          per batch) / their device time, in GB/s.
Extra keys: per-stage times, NTT GB/s, the roofline of the dominant kernel,
the config-1 encrypted training step (ms/step, replayed reference
train_iteration; decrypted weights vs the reference), config-3 bootstrapping
(ms, one CUDA graph), configs 4 / 5 (ms/step as the mean over their 8 / 5
steps: the recorded first step and the recorded steady-state second step,
decrypted weights vs the exact model), e2e through host buffers, the CPU
oracle baseline, clocks.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_LOG = 16
BATCH = 64
L_LIMBS = 24
DNUM = 3
W = 8


def c2_params(L):
    from paper_2506_19693_b200.scheme import make_params

    k = -(-40 * (-(-L // DNUM)) // 60)
    return make_params(level=L - 1, scale_bits=40, poly_degree=1 << N_LOG, first_bits=40,
                       special_bits=60 * k), k


def alg_bytes(L, k, batch, n_rot_keys):
    """BASELINE.md §3 (W=8): HMult (4l + 2b(l+k) + 2(l-1)) N W, HRot (4l + 2b(l+k)) N W,
    keys counted once per distinct key per batch."""
    n = 1 << N_LOG
    beta = DNUM
    key = 2 * beta * (L + k) * n * W
    hmult = batch * (4 * L + 2 * (L - 1)) * n * W + key
    hrot = batch * 4 * L * n * W + n_rot_keys * key
    ntt = 2 * (2 * batch * 2 * L * n * W)  # fwd + inv over both components
    return hmult, hrot, ntt


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            return None
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def pcie_probe(device_index: int, mb: int = 256, reps: int = 3) -> dict:
    """Raw pinned-memory copy rates of this box (H2D alone, D2H alone, both at once on two
    streams) and the GPU's PCIe link, so the end-to-end number can be read against the
    transfer floor of the box it ran on (boxes of this pool differ by up to 3x)."""
    import torch

    n = mb << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(up, dn):
        best = None
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s_up.wait_event(e0)
            s_dn.wait_event(e0)
            if up:
                with torch.cuda.stream(s_up):
                    d_in.copy_(h_in, non_blocking=True)
            if dn:
                with torch.cuda.stream(s_dn):
                    h_out.copy_(d_out, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s_up)
            torch.cuda.current_stream().wait_stream(s_dn)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return n * (int(up) + int(dn)) / (best / 1e3) / 1e9

    out = {"h2d_GBps": timed(True, False), "d2h_GBps": timed(False, True),
           "bidir_GBps": timed(True, True), "buffer_MB": mb}
    try:
        q = subprocess.run(
            ["nvidia-smi", "-i", str(device_index),
             "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max",
             "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
        g, w, gm = [int(x) for x in q.stdout.strip().split(",")]
        out["link"] = {"gen": g, "width": w, "gen_max": gm}
    except Exception:
        out["link"] = None
    return out


# ---------------------------------------------------------------------------
# CPU baselines (oracle port of the reference algorithm, reference prime layout)
# ---------------------------------------------------------------------------


def _cpu_case(L):
    from oracle import parallel_ref as PR

    return PR.make_random_case(1 << N_LOG, L, seed=5)


def _cpu_step(case, procs):
    """One HMult (mul + relinearise + rescale) and one HRot of one ciphertext
    with the reference's algorithm and prime layout (per-limb digits, sub-2^31
    primes; oracle/ckks_oracle.py), each key switch split over `procs` host
    processes (oracle/parallel_ref.py) — the B200 arm's step mix.  Returns
    seconds."""
    from oracle import parallel_ref as PR

    chain, (a, b), kb, ka = case
    _, s1 = PR.hmult_parallel(chain, a, b, kb, ka, procs)
    _, s2 = PR.hrot_parallel(chain, a, pow(5, 12345, 2 * chain.n), kb, ka, procs)
    return s1 + s2


def _cpu_sample_text(L, procs):
    return (f"one HMult + one HRot of one ciphertext (N=2^16, {L} x 40-bit entries in the "
            f"reference's sub-2^31 prime layout = {2 * L}+2 limbs, per-limb digits), numpy "
            f"oracle port of ckks/backend.py:136-171, key switch split over {procs} processes; "
            f"bytes = BASELINE HMult + HRot formulas at the B200 arm's parameters (1 key each)")


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port, numpy) on all
    host cores; one step = one HMult + one HRot of one ciphertext."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle import parallel_ref as PR

    L = args.limbs
    _, k = c2_params(L)
    hm, hr, _ = alg_bytes(L, k, 1, 1)
    procs = args.ref_procs or PR.default_procs()
    case = _cpu_case(L)
    times = []
    for step in range(args.warmup + args.steps):
        dt = _cpu_step(case, procs)
        if step >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = (hm + hr) / (ms / 1e3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": f"c2 HMult + HRot at N=2^16, L={L}: reference algorithm and "
                               f"prime layout on the host CPU", "batch_per_step": 1},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": procs, "kind": "port",
                         "sample": _cpu_sample_text(L, procs)},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


METRIC = "encrypted train ms/step; bootstrap ms; keyswitch GB/s vs HBM peak"


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def run_c1_train(device_index):
    """Config 1: the reference train_iteration's HE call sequence replayed on the
    B200 backend (BASELINE primes 1x60 + 8x40 + 1x60, HW-64 secret)."""
    import torch

    from paper_2506_19693_b200 import he_api
    from paper_2506_19693_b200.replay import Program
    from paper_2506_19693_b200.scheme import make_params

    path = os.path.join(ROOT, "tests", "golden", "c1_trace.npz")
    z = np.load(path)
    prog = Program.load(path)
    n, level, sb = (int(v) for v in z["params"])
    params = make_params(level=level, scale_bits=sb, poly_degree=n)
    t0 = time.perf_counter()
    cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3,
                         prime_layout="baseline", secret_hw=64)
    torch.cuda.synchronize()
    keygen_s = time.perf_counter() - t0
    env = prog.run(cust, 0, prog.n_setup)
    import itertools

    times = []
    first = None
    s0 = next(cust.backend._serials)  # serial counter after setup (peek, then restore)
    for rep in range(3):
        cust.backend._serials = itertools.count(s0)  # every repetition = the same step
        cust.backend._enc_cache.clear()  # ... and re-encodes its plaintexts, as a new step would
        e = dict(env)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e = prog.run(cust, prog.n_setup, None, e)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        first = first or e
    from paper_2506_19693_b200.executor import WaveExecutor

    ex = WaveExecutor(prog, cust)
    wtimes = []
    for rep in range(3):
        cust.backend._enc_cache.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ew = ex.run(dict(env), only_after_setup=True)
        torch.cuda.synchronize()
        wtimes.append(time.perf_counter() - t0)
    wb = np.stack([cust.backend._decrypt_values(ew[o]) for o in prog.outputs])
    # the same step as one CUDA graph (graphs.GraphedStep): every device op of
    # the step (encodes, encryptions, HE ops, update) replayed with one launch,
    # the host-round-trip refreshes eager afterwards
    from paper_2506_19693_b200.graphs import GraphedStep

    gs = GraphedStep(ex, env)
    gtimes = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eg = gs.step()
        torch.cuda.synchronize()
        gtimes.append(time.perf_counter() - t0)
    wg = np.stack([cust.backend._decrypt_values(eg[o]) for o in prog.outputs])
    from paper_2506_19693_b200.graphs import eager_equivalent

    ee = eager_equivalent(gs)  # the eager executor with the last replay's serials
    we = np.stack([cust.backend._decrypt_values(ee[o]) for o in prog.outputs])
    w = np.stack([cust.decrypt(first[o]).values for o in prog.outputs])
    err_sim = float(np.max(np.abs(w - z["sim_weights"])))
    err_ref = float(np.max(np.abs(w - z["ckks_weights"]))) if "ckks_weights" in z else None
    ref_s = float(z["ckks_seconds"][1]) if "ckks_seconds" in z else None
    return {"ms_per_step": 1e3 * min(gtimes), "ms_per_step_eager_waves": 1e3 * min(wtimes),
            "ms_per_step_sequential_api": 1e3 * min(times),
            "waves": len(ex.waves), "batched_weights_equal_sequential": bool(np.array_equal(wb, w)),
            "graph_weights_equal_eager_same_serials": bool(np.array_equal(wg, we)),
            "graph_weights_max_abs_diff_vs_sequential": float(np.max(np.abs(wg - w))),
            "timing": "ms_per_step: the step as one CUDA graph replay (all device work, "
                      "re-encoding every plaintext) + the 4 debug refreshes eager; wall clock "
                      "with a device sync on both sides",
            "ops": len(prog.ops) - prog.n_setup,
            "keygen_s": keygen_s, "weights_max_abs_err_vs_sim": err_sim,
            "weights_max_abs_err_vs_reference_ckks": err_ref,
            "reference_cpu_s_per_step_build_container": ref_s}


def run_c1_dropin(cpu: bool = True) -> dict:
    """Config 1 through the UNCHANGED reference layer code (tools/c1_dropin.py:
    the reference package from baseline/_ref — keygen, build_model,
    prepare_sample, nn.train_iteration — with plugin.install routing
    backend="ckks" to the B200 backend at the BASELINE primes), and the
    reference's own numpy CkksBackend timed on this host in the same run."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import c1_dropin as C

    C.import_reference()
    from paper_2506_19693_b200 import plugin

    gold = np.load(os.path.join(ROOT, "tests", "golden", "c1_modeA_weights.npy"))

    def timed(**opts):
        cls, old = plugin.install(prime_layout="baseline", secret_hw=64, **opts)
        try:
            times = []
            for rep in range(3):  # rep 0 warms tables / FFT plans
                cust, model, shape, x, onehot = C.build()
                cust.backend.flush()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                C.step(cust, model, shape, x, onehot)
                cust.backend.flush()
                torch.cuda.synchronize()
                times.append(time.perf_counter() - t0)
            return times, C.weights(model, cust)
        finally:
            plugin.uninstall(old)

    t_eager, w_eager = timed()
    t_def, w_def = timed(deferred=True)
    out = {"ms_per_step": 1e3 * min(t_def[1:]), "ms_per_step_eager_calls": 1e3 * min(t_eager[1:]),
           "first_step_ms": 1e3 * t_def[0],
           "weights_max_abs_err_vs_reference_ckks": float(np.max(np.abs(w_def - gold))),
           "deferred_weights_equal_eager": bool(np.array_equal(w_def, w_eager)),
           "path": "reference nn.train_iteration + prepare_sample (32 samples encrypted) through "
                   "ciphermlp.api -> plugin-installed B200 CkksBackend; ms_per_step: deferred "
                   "mode (the step's HE calls recorded and run as batched waves on the first "
                   "decrypt); ms_per_step_eager_calls: one HE call at a time",
           "timing": "wall clock from the first encryption to the refreshed weights on the "
                     "device (flush + sync), best of 2 after a warm-up step"}
    if cpu:
        ref = C.time_reference_step((1, 2))
        out["cpu_reference"] = ref
        out["speedup_vs_cpu_reference"] = ref["ms_per_step_batch32"] / out["ms_per_step"]
    return out


def run_c4_dp(local: int, world: int, reps: int = 3) -> dict:
    """Config 4's recorded step (tests/golden/c4_trace.npz: 128 samples, real
    bootstrapping) sharded by sample across `world` ranks (dp.py): per-sample
    pipelines on their owner, one exact residue all-reduce of the delta-W folds
    (NCCL), the update and the 4 bootstraps replicated.  Strong scaling (the
    batch of 128 is fixed); CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2506_19693_b200 import dist as hdist
    from paper_2506_19693_b200 import he_api
    from paper_2506_19693_b200.dp import DataParallelExecutor
    from paper_2506_19693_b200.replay import Program
    from paper_2506_19693_b200.scheme import SchemeParams

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import c4_run

    path = os.path.join(ROOT, "tests", "golden", "c4_trace.npz")
    z = np.load(path)
    prog = Program.load(path)
    n, L, sb, bd = (int(v) for v in z["params"])
    params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,),
                          scale_bits=45, level=L, bootstrap_depth=bd)
    cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=4,
                         prime_layout="bootstrap", dnum=3, secret_hw=192, real_bootstrap=True,
                         low_special=c4_run.LOW_SPECIAL)
    cust.backend.prepare_bootstrap()
    env = prog.run(cust, 0, prog.n_setup)
    ex = DataParallelExecutor(prog, cust, encs_per_sample=3)
    times = []
    out = None
    for rep in range(reps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cust.backend._enc_cache.clear()
        a.record()
        out = ex.run(dict(env), only_after_setup=True)
        b.record()
        torch.cuda.synchronize()
        dist.barrier()
        if rep:
            times.append(hdist.max_over_ranks(a.elapsed_time(b)))
    w = np.stack([cust.backend._decrypt_values(out[o]) for o in prog.outputs])
    planes = np.concatenate([cust.backend.planes_of(out[o]).ravel() for o in prog.outputs])
    digest = int(np.bitwise_xor.reduce(planes.view(np.int64)))
    lo = hdist.reduce_scalar(digest, dist.ReduceOp.MIN, torch.int64)
    hi = hdist.reduce_scalar(digest, dist.ReduceOp.MAX, torch.int64)
    return {"ms_per_step": min(times), "ranks": world, "scaling": "strong",
            "samples": ex.plan.n_samples,
            "samples_per_rank": len(hdist.shard(ex.plan.n_samples, dist.get_rank(), world)),
            "weights_identical_across_ranks": bool(lo == hi),
            "weights_max_abs_err_vs_sim": float(np.max(np.abs(w[:2] - z["sim_weights"][:2]))),
            "timing": "the recorded config-4 first step (4 real bootstraps), CUDA events around "
                      "the sharded step, max over ranks, best of 3 after a warm-up"}


def run_c1_dp(local: int, world: int) -> dict:
    """Config-1 step sharded by sample across `world` ranks (dp.py):
    each rank runs its share of the 32 per-sample pipelines, one exact residue
    all-reduce (NCCL int64 SUM + ckb_reduce) joins the δW partial sums, and the
    update + refresh run replicated.  Device-timed, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2506_19693_b200 import dist as hdist
    from paper_2506_19693_b200 import he_api
    from paper_2506_19693_b200.dp import DataParallelExecutor
    from paper_2506_19693_b200.replay import Program
    from paper_2506_19693_b200.scheme import make_params

    path = os.path.join(ROOT, "tests", "golden", "c1_trace.npz")
    z = np.load(path)
    prog = Program.load(path)
    n, level, sb = (int(v) for v in z["params"])
    params = make_params(level=level, scale_bits=sb, poly_degree=n)
    cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3,
                         prime_layout="baseline", secret_hw=64)
    env = prog.run(cust, 0, prog.n_setup)
    ex = DataParallelExecutor(prog, cust, encs_per_sample=3)
    times = []
    out = None
    for rep in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cust.backend._enc_cache.clear()
        a.record()
        out = ex.run(dict(env), only_after_setup=True)
        b.record()
        torch.cuda.synchronize()
        dist.barrier()
        if rep:  # first repetition = warm-up
            times.append(hdist.max_over_ranks(a.elapsed_time(b)))
    # every rank must hold the same refreshed weights
    planes = np.concatenate([cust.backend.planes_of(out[o]).ravel() for o in prog.outputs])
    digest = int(np.bitwise_xor.reduce(planes.view(np.int64)))
    lo = hdist.reduce_scalar(digest, dist.ReduceOp.MIN, torch.int64)
    hi = hdist.reduce_scalar(digest, dist.ReduceOp.MAX, torch.int64)
    return {"ms_per_step": min(times), "ranks": world, "samples": ex.plan.n_samples,
            "samples_per_rank": len(hdist.shard(ex.plan.n_samples, dist.get_rank(), world)),
            "allreduce_bytes_per_rank": ex.exchanged_bytes // len(range(4)),
            "weights_identical_across_ranks": bool(lo == hi),
            "timing": "CUDA events around the sharded step, max over ranks"}


def security_note(be) -> str:
    """HES gate of the chain actually built (params.py:70-77: 1,772 bits at N=2^16)."""
    bits = sum(int(p).bit_length() for p in be.chain.all_primes)
    bound = {2**12: 109, 2**13: 218, 2**14: 438, 2**15: 881, 2**16: 1772, 2**17: 3544}.get(
        be.n, 0)
    tag = "insecure-test" if bits > bound else "128-bit (HE standard)"
    return f"{tag}: log2(QP) = {bits} bits vs the {bound}-bit bound at N={be.n}"


def run_c3_bootstrap(special: int = 660):
    """Config 3: full-slot bootstrapping of one ciphertext at N=2^16 (2^15 slots,
    U[-1,1]), input at level 0, HW-192 secret, CtS/StC 3 BSGS levels each,
    EvalMod = degree-119 Chebyshev + 2 double-angle steps (bootstrap.py)."""
    import torch

    from paper_2506_19693_b200 import he_api
    from paper_2506_19693_b200.scheme import SchemeParams

    n, L = 1 << 16, 24
    params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (special,),
                          scale_bits=45, level=L, bootstrap_depth=16)
    t0 = time.perf_counter()
    cust = he_api.keygen(params, set(), backend="ckks", rng_seed=11, prime_layout="bootstrap",
                         dnum=3, secret_hw=192, real_bootstrap=True)
    be = cust.backend
    torch.cuda.synchronize()
    keygen_s = time.perf_counter() - t0
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, n // 2)
    ct = be._encrypt_values(v, 0)
    times = []
    out = None
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = be.bootstrap_ct(ct)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    err = float(np.max(np.abs(be._decrypt_values(out) - v)))
    # the same bootstrap as one CUDA graph replay (graphs.GraphedCall): the
    # input ciphertext is copied into the graph's static input every call
    from paper_2506_19693_b200.backend import GpuCiphertext
    from paper_2506_19693_b200.graphs import GraphedCall

    gc = GraphedCall(lambda d: be.bootstrap_ct(GpuCiphertext(d, 0)).data, ct.data)
    gtimes = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gc.load(ct.data)
        gout = gc()
        torch.cuda.synchronize()
        gtimes.append(time.perf_counter() - t0)
    graph_equal = bool(torch.equal(gout.view(torch.int64), out.data.view(torch.int64)))
    return {"ms": 1e3 * float(np.median(gtimes)), "ms_eager": 1e3 * float(np.median(times[1:])),
            "graph_output_equal_eager": graph_equal, "first_call_ms": 1e3 * times[0],
            "max_abs_err": err, "precision_bits": -math.log2(err), "level_out": out.level,
            "keys": len(be.rotation_keys) + 1, "keygen_s": keygen_s,
            "security": security_note(be),
            "params": "N=2^16, 2^15 slots, Q = 60 + 8x45 (user) + 16x60 (bootstrap) bits, "
                      "P = 11x60, dnum=3, HW 192, K=28, Chebyshev 119 + 2 double angles"}


def load_traffic() -> dict:
    """Per-launch DRAM traffic of the profiled kernels (ncu dram__bytes_read.sum +
    dram__bytes_write.sum), committed under profiles/ from the capture named in
    each entry's "source"."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


TRAFFIC = load_traffic()


def alu_probe_gbfly(p: int, reps: int = 3, f64: bool = False) -> float:
    """Peak lazy-CT-butterfly rate (G butterflies/s) of the IMAD/ALU pipes,
    register-resident (ckb_alu_probe): the NTT's binding roofline."""
    import torch

    from paper_2506_19693_b200 import _native as nat

    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 16, 1000
    w = (p * 2) // 3
    fn = nat.LIB.ckb_alu_probe_f64 if f64 else nat.LIB.ckb_alu_probe
    nat.check(fn(p, w, 10, blocks, nat.ptr(sink), nat.stream_handle()), "probe")
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nat.check(fn(p, w, iters, blocks, nat.ptr(sink), nat.stream_handle()), "probe")
        b.record()
        torch.cuda.synchronize()
        best = max(best, blocks * 256 * 12 * iters / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def tc_probe_gmacs(reps: int = 3) -> float:
    """Measured u8 MAC rate (G MAC/s) of the tensor pipes: every SM issuing
    back-to-back tcgen05.mma kind::i8 M=128 N=256 K=32 (ckb_tc_probe): the
    roofline of the basis-conversion GEMMs (csrc/tc.cu)."""
    import torch

    from paper_2506_19693_b200 import _native as nat

    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ctas, iters = sms * 2, 4000
    nat.check(nat.LIB.ckb_tc_probe(ctas, 10, nat.ptr(sink), nat.stream_handle()), "tc_probe")
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nat.check(nat.LIB.ckb_tc_probe(ctas, iters, nat.ptr(sink), nat.stream_handle()),
                  "tc_probe")
        b.record()
        torch.cuda.synchronize()
        best = max(best, ctas * iters * (1 << 20) / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def cpu_reference(L, args) -> dict:
    """The reference algorithm (oracle port, its own prime layout) on this
    host's cores: one HMult + one HRot of one ciphertext at N=2^16, L entries."""
    from oracle import parallel_ref as PR

    procs = args.ref_procs or PR.default_procs()
    secs = _cpu_step(_cpu_case(L), procs)
    _, k = c2_params(L)
    hm1, hr1, _ = alg_bytes(L, k, 1, 1)
    return {"value": (hm1 + hr1) / secs / 1e9, "unit": "GB/s", "cores": procs, "kind": "port",
            "seconds": secs, "sample": _cpu_sample_text(L, procs)}


def pair_alu_floor(be, L, k, bsz, peak_int, peak_f64, peak_tc=None):
    """Arithmetic floor of one HMult batch + one HRot batch (the headline pair):
    every modular multiply the algorithm needs — NTT butterflies (N/2 log N per
    limb transform), the ModUp premultiplies y_i, inner-product MACs (2 per
    digit per ext limb), the ModDown y_u, tensor products (4) and combine
    multiplies (2) — each charged to the FP64 (primes < 2^46) or integer
    (60-bit) pipe by its prime and timed at that pipe's measured butterfly rate
    (ckb_alu_probe / ckb_alu_probe_f64; a butterfly is one modular multiply
    plus an add and a subtract).  The basis conversions (ModUp's per-output
    sums over the digit, the ModDown correction's sums over the dropped primes)
    run on the tensor cores when the chain sets CKB_RING_TC: their u8 MACs
    (8 value bytes x 5 or 8 constant bytes per term) are timed at the measured
    tensor-pipe rate (ckb_tc_probe) and their per-output reductions at the
    integer rate; without the tensor cores every term is a CUDA-core modular
    multiply.  Pipes are summed (no overlap credited); memory traffic is free."""
    n = 1 << N_LOG
    bf = n // 2 * N_LOG  # butterflies per limb transform
    alpha = -(-L // DNUM)
    nd = -(-L // alpha)
    m = L
    m2 = m - 1
    tc = peak_tc is not None
    nb = lambda wide: 8 if wide else 5  # noqa: E731  (config 2: 40-bit Q, 60-bit P)
    acc = {"f": 0, "i": 0, "t": 0}

    def modup():
        for j in range(nd):
            cnt = min(alpha, m - j * alpha)
            acc["f"] += cnt * n + (m - cnt) * bf
            acc["i"] += k * bf
            if tc:
                acc["t"] += n * cnt * 8 * ((m - cnt) * nb(False) + k * nb(True))
                acc["i"] += (m - cnt + k) * n
            else:
                acc["f"] += (m - cnt) * cnt * n
                acc["i"] += k * cnt * n
        acc["f"] += 2 * nd * m * n          # inner product, Q limbs
        acc["i"] += 2 * nd * k * n          # inner product, P limbs

    def moddown(kept, n2):
        acc["i"] += 2 * (k + n2) * bf + 2 * (k + n2) * n  # iNTT of dropped limbs, their y_u
        if tc:
            nvals = k + 1 + n2
            acc["t"] += 2 * n * kept * nvals * 8 * nb(False)
            acc["i"] += 2 * kept * n
        else:
            acc["f"] += 2 * kept * (k + n2) * n
        acc["f"] += 2 * (kept * bf + 2 * kept * n)      # NTT of E, combine

    # HMult: tensor, iNTT(d2), ModUp, NTT(digits), inner product, ModDown + rescale
    acc["f"] += 4 * m * n + m * bf
    modup()
    moddown(m2, 1)
    # HRot: automorphism (a permutation), iNTT(c1'), ModUp, NTT, MAC, ModDown
    acc["f"] += m * bf
    modup()
    moddown(m, 0)
    tot_f = bsz * acc["f"] / 1e9
    tot_i = bsz * acc["i"] / 1e9
    tot_t = bsz * acc["t"] / 1e9
    floor_s = tot_f / peak_f64 + tot_i / peak_int + (tot_t / peak_tc if tc else 0.0)
    return {"gmulmod_f64": tot_f, "gmulmod_int": tot_i, "gmac_u8_tensor": tot_t,
            "floor_ms": 1e3 * floor_s, "peak_int_gbfly": peak_int, "peak_f64_gbfly": peak_f64,
            "peak_tc_gmacs": peak_tc, "tensor_cores": tc}


def run_c2(L, bsz, args, rank, world, local, breakdown=False, keep=False) -> dict:
    """One BASELINE config-2 point: keys, a 64-ciphertext batch, the HMult + HRot
    pair on two streams timed with CUDA events (max over ranks), optionally the
    sequential per-stage / per-kernel breakdown and the rooflines."""
    import torch

    from paper_2506_19693_b200 import dist as hdist
    from paper_2506_19693_b200 import he_api, ring
    from paper_2506_19693_b200.ring import KernelTimer

    params, k = c2_params(L)
    rng = np.random.default_rng(1234 + rank)
    steps_rot = [int(s) for s in rng.integers(1, 1 << 15, bsz)]
    t0 = time.perf_counter()
    cust = he_api.keygen(params, set(steps_rot), backend="ckks", rng_seed=99 + rank,
                         prime_layout="baseline", dnum=DNUM, secret_hw=192)
    be = cust.backend
    torch.cuda.synchronize()
    keygen_s = time.perf_counter() - t0
    lvl = params.level
    m = be.chain.level_limbs[lvl]
    n = 1 << N_LOG
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7 + rank)

    def rand_batch():
        t = torch.empty(bsz, 2, m, n, dtype=torch.int64, device="cuda")
        for i, p in enumerate(be.chain.limbs_at(lvl)):
            t[:, :, i].random_(0, p, generator=gen)
        return t.view(torch.uint64)

    A, B = rand_batch(), rand_batch()
    X = torch.empty_like(A)
    slots = params.slot_count
    n_keys = len({s % slots for s in steps_rot})  # distinct Galois keys of the HRot batch
    hm_b, hr_b, ntt_b = alg_bytes(L, k, bsz, n_keys)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    s_hm, s_hr = torch.cuda.Stream(), torch.cuda.Stream()

    def keyswitch_pair():
        # the HMult and HRot batches are independent: two streams (their
        # kernels are bound by different resources and overlap); each stream's
        # transforms get half the single-stream L2 budget (ckb_ring)
        cur = torch.cuda.current_stream()
        s_hm.wait_stream(cur)
        s_hr.wait_stream(cur)
        prev = be.chain.set_ntt_chunk_bytes(48 << 20)
        try:
            with torch.cuda.stream(s_hm):
                be.batch_hmult(A, B, lvl)
            with torch.cuda.stream(s_hr):
                be.batch_hrot(A, steps_rot, lvl)
        finally:
            be.chain.set_ntt_chunk_bytes(prev)
        cur.wait_stream(s_hm)
        cur.wait_stream(s_hr)

    for _ in range(args.warmup):
        X.copy_(A)
        be.batch_ntt(X, lvl)
        be.batch_ntt(X, lvl, inverse=True)
        keyswitch_pair()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    pairs = []
    start, end = ev(), ev()
    torch.cuda.synchronize()
    start.record()
    for _ in range(args.steps):
        e1, e2 = ev(), ev()
        X.copy_(A)
        be.batch_ntt(X, lvl)
        be.batch_ntt(X, lvl, inverse=True)
        e1.record()
        keyswitch_pair()
        e2.record()
        pairs.append((e1, e2))
    end.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms_step = hdist.max_over_ranks(start.elapsed_time(end)) / args.steps
    ks_ms = hdist.max_over_ranks(float(np.mean([a.elapsed_time(b) for a, b in pairs])))
    value = world * (hm_b + hr_b) / (ks_ms / 1e3) / 1e9  # weak scaling: every rank its batch
    out = {"value": value, "ms_per_step": ms_step, "keyswitch_pair_ms": ks_ms, "L": L, "k": k,
           "alpha": be.alpha, "batch": bsz, "distinct_rotation_keys": n_keys,
           "alg_bytes": {"hmult": hm_b, "hrot": hr_b, "ntt_intt": ntt_b},
           "keygen_s": keygen_s,
           "timing": "value: HMult and HRot batches on two streams, CUDA events around the "
                     "pair, mean over steps, max over ranks" +
                     ("; stages_ms / kernels / roofline: a second pass of the same steps "
                      "issued sequentially with events around every kernel" if breakdown else "")}
    if clk:
        out["clocks"] = clk
    if breakdown:
        timer = KernelTimer()
        ring.TIMER = timer
        stage = {"ntt": [], "hmult": [], "hrot": []}
        torch.cuda.synchronize()
        for _ in range(args.steps):
            e0, e1, e2, e3 = ev(), ev(), ev(), ev()
            e0.record()
            X.copy_(A)
            be.batch_ntt(X, lvl)
            be.batch_ntt(X, lvl, inverse=True)
            e1.record()
            be.batch_hmult(A, B, lvl)
            e2.record()
            be.batch_hrot(A, steps_rot, lvl)
            e3.record()
            stage["ntt"].append((e0, e1))
            stage["hmult"].append((e1, e2))
            stage["hrot"].append((e2, e3))
        torch.cuda.synchronize()
        ring.TIMER = None
        # median over the steps (a rare stall of one step would skew a mean);
        # the spread is reported beside it
        st_all = {kk: [a.elapsed_time(b) for a, b in v] for kk, v in stage.items()}
        st_ms = {kk: float(np.median(v)) for kk, v in st_all.items()}
        out["stages_ms_minmax"] = {kk: [float(min(v)), float(max(v))] for kk, v in st_all.items()}
        ksum = timer.summary()
        launches = sum(d["launches"] for d in ksum.values())
        dom_name = max(ksum, key=lambda nm: ksum[nm]["ms"])
        dom = ksum[dom_name]
        peak, peak_kind = load_peaks()
        achieved = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
        out["stages_ms"] = st_ms
        out["hmult_GBps"] = hm_b / (st_ms["hmult"] / 1e3) / 1e9
        out["hrot_GBps"] = hr_b / (st_ms["hrot"] / 1e3) / 1e9
        out["ntt_GBps"] = ntt_b / (st_ms["ntt"] / 1e3) / 1e9
        out["hmult_us_per_ct"] = 1e3 * st_ms["hmult"] / bsz
        out["hrot_us_per_ct"] = 1e3 * st_ms["hrot"] / bsz
        out["kernels"] = {nm: {"ms_per_step": d["ms"] / args.steps,
                               "launches_per_step": d["launches"] / args.steps,
                               "GBps_alg": d["bytes"] / (d["ms"] / 1e3) / 1e9,
                               "share": d["ms"] / sum(x["ms"] for x in ksum.values())}
                          for nm, d in ksum.items()}
        out["gpu_launches"] = launches
        out["roofline"] = {"bound": "hbm", "kernel": dom_name, "achieved": achieved,
                           "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                           "frac": achieved / peak,
                           "traffic": (TRAFFIC.get(dom_name) or {}).get("dram_bytes_per_launch"),
                           "traffic_detail": TRAFFIC.get(dom_name)}
        p_int = int(be.chain.special_primes[0])  # a 60-bit special prime
        p_f64 = int(be.chain.limbs_at(lvl)[-1])  # a 40-bit Q prime
        peak_int = alu_probe_gbfly(p_int)
        peak_f64 = alu_probe_gbfly(p_f64, f64=True)
        if dom_name in ("ntt", "intt", "ntt_combine"):
            # the NTT's binding roofline is the arithmetic pipes, not HBM: rows
            # with primes < 2^46 run the FP64 butterfly, the others the integer
            # one, each against its own register-resident probe
            bf = dom["bytes"] * N_LOG / 32 / 1e9          # G butterflies (bytes = 16 N per limb)
            bf_f64 = dom["f64_bytes"] * N_LOG / 32 / 1e9
            floor_s = (bf - bf_f64) / peak_int + bf_f64 / peak_f64
            got_s = dom["ms"] / 1e3
            out["roofline"]["alu"] = {
                "unit": "Gbutterfly/s", "achieved": bf / got_s, "peak": bf / floor_s,
                "frac": floor_s / got_s, "f64_share": bf_f64 / bf, "peak_int": peak_int,
                "peak_f64": peak_f64,
                "peak_source": "ckb_alu_probe / ckb_alu_probe_f64 (register-resident "
                               "butterflies, the NTT's own integer and FP64 arithmetic), "
                               "weighted by this kernel's row mix"}
        from paper_2506_19693_b200 import _native as nat_

        use_tc = bool(be.chain.ring.flags & nat_.RING_TC)
        fl = pair_alu_floor(be, L, k, bsz, peak_int, peak_f64,
                            tc_probe_gmacs() if use_tc else None)
        seq_ms = st_ms["hmult"] + st_ms["hrot"]
        out["pair_roofline"] = {
            "alu_floor_ms": fl["floor_ms"], "hbm_floor_ms": 1e3 * (hm_b + hr_b) / peak / 1e9,
            "pair_ms": ks_ms, "sequential_ms": seq_ms, "alu_frac": fl["floor_ms"] / ks_ms,
            "hbm_frac": (hm_b + hr_b) / (ks_ms / 1e3) / 1e9 / peak, **fl,
            "model": pair_alu_floor.__doc__.split("\n\n")[0].replace("\n", " ")}
    if keep:
        out["_live"] = (be, A, B, steps_rot, lvl, hm_b, hr_b)
    else:
        del A, B, X, cust, be
    return out


def e2e_he_api(be, A, B, steps_rot, lvl, hm_b, hr_b, world, reps=2) -> dict:
    """The c2 pair through the public HE API one ciphertext at a time, host
    bytes in and out: RBCT blobs (ckks/backend.py:210-247) -> deserialize_cipher
    (H2D + NTT) -> Evaluator.mul / Evaluator.rotate (the reference's
    api.py:270-294 calls, level/depth bookkeeping included) -> serialize_cipher
    (iNTT + D2H) for all 64 pairs; wall clock with a device sync at both ends."""
    import torch

    from paper_2506_19693_b200 import he_api
    from paper_2506_19693_b200.backend import GpuCiphertext

    cust = he_api.KeyCustodian(be, be.rotation_indices)
    evl = cust.evaluator
    bsz = A.shape[0]

    def wrap(d):
        return be._wrap(GpuCiphertext(d, lvl), lvl, 0)

    blobs_a = [be.serialize_cipher(wrap(A[i])) for i in range(bsz)]
    blobs_b = [be.serialize_cipher(wrap(B[i])) for i in range(bsz)]
    slots = be.params.slot_count

    def step():
        out = []
        for i in range(bsz):
            ca, cb = be.deserialize_cipher(blobs_a[i]), be.deserialize_cipher(blobs_b[i])
            out.append(be.serialize_cipher(evl.mul(ca, cb)))
            out.append(be.serialize_cipher(evl.rotate(ca, steps_rot[i] % slots)))
        return out

    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        res = step()
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0) / reps
    h2d = sum(len(b) for b in blobs_a) + sum(len(b) for b in blobs_b)
    d2h = sum(len(b) for b in res)
    return {"value": world * (hm_b + hr_b) / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "per-ciphertext HE API: RBCT bytes -> deserialize_cipher -> Evaluator.mul / "
                    "Evaluator.rotate -> serialize_cipher, 64 pairs, wall clock"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--limbs", type=int, default=L_LIMBS)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c1", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--ref-procs", type=int, default=0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2506_19693_b200 import he_api, ring
    from paper_2506_19693_b200.ring import KernelTimer

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CKB_SAME_DEVICE / CKB_DIST_BACKEND: functional check of the N>1 code path
    # on a one-GPU box (all ranks on cuda:0, exchange over gloo); never a bench number
    if os.environ.get("CKB_SAME_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("CKB_DIST_BACKEND", "nccl")
        # NCCL's own log (stderr) records the communicator's rank count and
        # transport (NVLink / NVLS) for the driver's checks
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2506_19693_b200 import dist as hdist

    L, bsz = args.limbs, args.batch
    head = run_c2(L, bsz, args, rank, world, local, breakdown=True, keep=True)
    be, A, B, steps_rot, lvl, hm_b, hr_b = head.pop("_live")
    line = {
        "metric": METRIC, "value": head["value"], "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": f"c2 primitive sweep: N=2^16, L={L} x 40-bit, dnum={DNUM}, "
                               f"k={head['k']} x 60-bit special, batch {bsz} ct: NTT+iNTT, "
                               f"HMult, HRot ({head['distinct_rotation_keys']} distinct keys)",
                   "batch_per_gpu": bsz, "l2": "inputs 1.5 GiB per operand > 126 MB L2 (no flush)",
                   "parallelism": f"replicas x{world} (independent ciphertext batches)"},
    }
    line.update({kk: v for kk, v in head.items() if kk not in ("value", "ms_per_step")})
    m = be.chain.level_limbs[lvl]
    n = 1 << N_LOG
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    if not args.no_e2e:
        line["e2e_he_api"] = e2e_he_api(be, A, B, steps_rot, lvl, hm_b, hr_b, world)
    if not args.no_e2e:
        # e2e: host (pinned) inputs -> device -> HMult + HRot -> host, per step.
        # The host batches are in the packed transfer format (backend.pack_batch:
        # 5 bytes per 40-bit residue instead of 8), unpacked / packed on the
        # device inside the timed region: PCIe carries 5/8 of the u64 bytes.
        lvl_out = lvl - 1
        hA = be.pack_batch(A, lvl).cpu().pin_memory()
        hB = be.pack_batch(B, lvl).cpu().pin_memory()
        nb_m = be.chain.packed_bytes(2, be.chain.level_limbs[lvl_out])
        nb_r = be.chain.packed_bytes(2, m)
        hOm = torch.empty(bsz, nb_m, dtype=torch.uint8).pin_memory()
        hOr = torch.empty(bsz, nb_r, dtype=torch.uint8).pin_memory()

        from paper_2506_19693_b200.streaming import Pipeline

        pipe = Pipeline()
        # 16 chunks when each chunk replays as a CUDA graph (below); eager calls use 8: 16 chunks
        # are ~4,400 kernel launches per step and host-enqueue-bound on this pool's slower hosts
        use_graphs = os.environ.get("CKB_E2E_GRAPHS", "1") != "0"
        chunk = int(os.environ.get("CKB_E2E_CHUNK", "0")) or max(1, bsz // (16 if use_graphs else 8))

        def e2e_chunk(dev, lo, hi):
            a = be.unpack_batch(dev[0], lvl)
            b = be.unpack_batch(dev[1], lvl)
            return [be.pack_batch(be.batch_hmult(a, b, lvl), lvl_out),
                    be.pack_batch(be.batch_hrot(a, steps_rot[lo:hi], lvl), lvl)]

        # One CUDA graph per chunk (its rotation steps and key pointers are fixed): the
        # chunk's ~280 kernel launches replay as one, so the step is no longer bound by the
        # host's enqueue rate (eager: 2,200 launches per step in 8 chunks, 64 ms on this pool's
        # slower hosts against a 40 ms PCIe floor).  CKB_E2E_GRAPHS=0 keeps the eager calls.
        graphs, graph_err = None, None
        if use_graphs:
            try:
                from paper_2506_19693_b200.graphs import GraphedCall

                graphs = []
                for lo in range(0, bsz, chunk):
                    hi = min(bsz, lo + chunk)
                    graphs.append(GraphedCall(
                        lambda a, b, lo=lo, hi=hi: e2e_chunk([a, b], lo, hi),
                        hA[lo:hi].to("cuda"), hB[lo:hi].to("cuda"), warmup=1))
            except Exception as exc:  # report, never hide; the eager path still runs
                graphs, graph_err = None, repr(exc)
                torch.cuda.synchronize()
                chunk = int(os.environ.get("CKB_E2E_CHUNK", "0")) or max(1, bsz // 8)

        def e2e_chunk_graph(dev, lo, hi):
            g = graphs[lo // chunk]
            g.load(*dev)  # device-to-device into the graph's static inputs
            return g()    # (its static outputs are read by this step's D2H copy, which the
                          #  step's final join orders before the next step's replay)

        def e2e_step():  # H2D / unpack, HMult+HRot, pack / D2H overlapped across chunks
            pipe.run(e2e_chunk_graph if graphs else e2e_chunk, [hA, hB], [hOm, hOr], chunk)

        e2e_step()
        torch.cuda.synchronize()
        # the round trip is exact: the unpacked HMult output equals the batch call's
        chk = be.unpack_batch(hOm[:chunk].to("cuda"), lvl_out)
        ok = torch.equal(chk.view(torch.int64),
                         be.batch_hmult(A[:chunk], B[:chunk], lvl).view(torch.int64))
        lo_l = ((bsz - 1) // chunk) * chunk  # ... and the last chunk's rotations
        chk = be.unpack_batch(hOr[lo_l:].to("cuda"), lvl)
        ok = ok and torch.equal(chk.view(torch.int64),
                                be.batch_hrot(A[lo_l:], steps_rot[lo_l:], lvl).view(torch.int64))
        s0, s1 = ev(), ev()
        s0.record()
        e2e_reps = max(4, args.steps)
        for _ in range(e2e_reps):
            e2e_step()
        s1.record()
        torch.cuda.synchronize()
        e2e_ms = hdist.max_over_ranks(s0.elapsed_time(s1)) / e2e_reps
        line["e2e"] = {"value": world * (hm_b + hr_b) / (e2e_ms / 1e3) / 1e9, "unit": "GB/s",
                       "ms_per_step": e2e_ms, "pipelined_chunks": -(-bsz // chunk),
                       "h2d_bytes_per_step": hA.numel() + hB.numel(),
                       "d2h_bytes_per_step": hOm.numel() + hOr.numel(),
                       "transfer_format": "packed residues (ckb_pack: 5 bytes per 40-bit "
                                          "residue), unpacked/packed on the device in the "
                                          "timed region",
                       "cuda_graphs": bool(graphs), "output_equal_batch_call": bool(ok)}
        if graph_err:
            line["e2e"]["cuda_graphs_error"] = graph_err
        graphs = None
        del hA, hB, hOm, hOr
        try:  # the box's own PCIe floor for these bytes, beside the number it bounds
            pc = pcie_probe(local)
            moved = line["e2e"]["h2d_bytes_per_step"] + line["e2e"]["d2h_bytes_per_step"]
            pc["floor_ms"] = moved / (pc["bidir_GBps"] * 1e9) * 1e3
            pc["frac"] = pc["floor_ms"] / e2e_ms
            line["e2e"]["pcie"] = pc
        except Exception as exc:  # report, never hide
            line["e2e"]["pcie"] = {"error": repr(exc)}

    del A, B
    torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not args.no_c1:
        try:
            line["c1_train"] = run_c1_train(local)
        except Exception as exc:  # report, never hide
            line["c1_train"] = {"error": repr(exc)}
        try:
            line["c1_train_dropin"] = run_c1_dropin(cpu=not args.no_cpu)
        except Exception as exc:  # report, never hide
            line["c1_train_dropin"] = {"error": repr(exc)}
    if world > 1 and not args.no_c1:
        try:
            res = run_c1_dp(local, world)
        except Exception as exc:
            res = {"error": repr(exc)}
        if rank == 0:
            line["c1_train_dp"] = res
    if world > 1 and not args.no_c4:
        try:
            torch.cuda.empty_cache()
            res = run_c4_dp(local, world)
        except Exception as exc:
            res = {"error": repr(exc)}
        if rank == 0:
            line["c4_train_dp"] = res
    if rank == 0 and world == 1 and not args.no_c3:
        try:
            line["c3_bootstrap"] = run_c3_bootstrap()
        except Exception as exc:
            line["c3_bootstrap"] = {"error": repr(exc)}
    # configs 4 and 5: every step executed through the unchanged reference layer
    # code (tools/train_dropin.py), weights checked against the simulator
    for cname, skip in (("c4", args.no_c4), ("c5", args.no_c5)):
        if rank == 0 and world == 1 and not skip:
            try:
                import gc as _gc

                _gc.collect()  # earlier legs' backends (reference cycles) and graph pools
                torch.cuda.empty_cache()
                sys.path.insert(0, os.path.join(ROOT, "tools"))
                import train_dropin

                line[f"{cname}_train"] = train_dropin.run(cname)
            except Exception as exc:
                line[f"{cname}_train"] = {"error": repr(exc)}
            torch.cuda.empty_cache()
    if not args.no_sweep:
        # BASELINE config 2's other limb counts, each a full c2 step of its own
        # (keys, batch, two-stream pair timing) with the CPU reference at that L
        sweep = {}
        for Ls in (4, 12):
            if Ls == L:
                continue
            try:
                r = run_c2(Ls, bsz, args, rank, world, local, breakdown=False)
                if rank == 0 and world == 1 and not args.no_cpu:
                    r["cpu_reference"] = cpu_reference(Ls, args)
                    r["speedup_vs_cpu_reference"] = r["value"] / r["cpu_reference"]["value"]
                sweep[f"L{Ls}"] = r
            except Exception as exc:  # report, never hide
                sweep[f"L{Ls}"] = {"error": repr(exc)}
            torch.cuda.empty_cache()
        line["c2_sweep"] = sweep
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_reference(L, args)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
