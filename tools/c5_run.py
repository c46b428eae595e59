"""Config 5 (deep tabular): 64->64->64->64->64->2, batch 256,
N=2^16, L = 16 user + 16 bootstrap levels (insecure-test), 16 real bootstraps
per step: the reference train_iteration's HE calls (tests/golden/c5_trace.npz),
wave-batched in sub-batches of `max_group` ciphertexts."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import SchemeParams


# training-step key switches over Q u P' with P' the first special primes above
# the widest digit of the level (backend.B200CkksCore low_special): levels <= 16 (digits <= 510 bits) over 9 x 60-bit special primes, levels
# 17..32 (digits <= 660 bits) over 12;
# bootstrapping keeps the full P
LOW_SPECIAL = [(16, 9), (32, 12)]

def run(reps=1, max_group=64, verbose=True, special=780, graph=True):
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                        "golden", "c5_trace.npz")
    z = np.load(path); prog = Program.load(path)
    n, L, sb, bd = (int(v) for v in z["params"])
    user = L - bd
    # P = 13 x 60 bits: 120 bits above the widest digit (11 x 60-bit bootstrap primes)
    params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * user + (60,) * bd + (special,),
                          scale_bits=45, level=L, bootstrap_depth=bd)
    t0 = time.perf_counter()
    cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=5,
                         prime_layout="bootstrap", dnum=3, secret_hw=192, real_bootstrap=True,
                         low_special=LOW_SPECIAL)
    torch.cuda.synchronize(); keygen_s = time.perf_counter() - t0
    env = prog.run(cust, 0, prog.n_setup)
    ex = WaveExecutor(prog, cust, max_group=max_group)
    times = []
    out = None
    for rep in range(reps):
        torch.cuda.reset_peak_memory_stats()
        cust.backend._enc_cache.clear()  # every step re-encodes its plaintexts
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = ex.run(dict(env), only_after_setup=True)
        torch.cuda.synchronize(); times.append(time.perf_counter() - t0)
        if verbose:
            print(f"step {rep}: {times[-1]*1e3:.1f} ms, peak mem "
                  f"{torch.cuda.max_memory_allocated()/2**30:.1f} GiB", flush=True)
    w = np.stack([cust.backend._decrypt_values(out[o]) for o in prog.outputs])
    ref = z["sim_weights"]
    err = np.max(np.abs(w - ref), axis=1)
    mag = np.max(np.abs(ref), axis=1)
    kind = np.arange(len(prog.outputs)) % 4  # per block: layer w, classifier w, velocities
    # steady state: the trace's second train_iteration on step 1's refreshed state
    prog2 = Program.load_step2(path)
    env2 = {k: out[k] for k in prog.keep}
    del out
    ex2 = WaveExecutor(prog2, cust, max_group=max_group)
    t2 = []
    for rep in range(reps):
        cust.backend._enc_cache.clear()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out2 = ex2.run(dict(env2), only_after_setup=True)
        torch.cuda.synchronize(); t2.append(time.perf_counter() - t0)
        if verbose:
            print(f"steady step {rep}: {t2[-1]*1e3:.1f} ms", flush=True)
    w2 = np.stack([cust.backend._decrypt_values(out2[o]) for o in prog2.outputs])
    err2 = np.max(np.abs(w2 - z["sim_weights_step2"]), axis=1)
    step1_ms, step2_ms = 1e3 * min(times), 1e3 * min(t2)
    step2_eager_ms, graph_equal, graph_err = step2_ms, None, None
    if graph:  # the steady step (smaller than step 1) as one CUDA graph
        del out2
        torch.cuda.empty_cache()
        try:
            from paper_2506_19693_b200.graphs import GraphedStep

            gs2 = GraphedStep(ex2, env2, warmup=1)
            g2 = []
            for rep in range(max(reps, 2)):
                torch.cuda.synchronize(); t0 = time.perf_counter()
                og2 = gs2.step()
                torch.cuda.synchronize(); g2.append(time.perf_counter() - t0)
            wg2 = np.stack([cust.backend._decrypt_values(og2[o]) for o in prog2.outputs])
            from paper_2506_19693_b200.graphs import eager_equivalent
            oe2 = eager_equivalent(gs2)
            graph_equal = bool(np.array_equal(wg2, np.stack([cust.backend._decrypt_values(oe2[o]) for o in prog2.outputs])))
            step2_ms = 1e3 * min(g2)
            del gs2, og2
        except torch.OutOfMemoryError as exc:  # keep the eager number
            graph_err = repr(exc)[:200]
        torch.cuda.empty_cache()
    return {"ms_per_step": (step1_ms + 4 * step2_ms) / 5, "steps": 5, "step1_ms": step1_ms,
            "steady_step_ms": step2_ms, "steady_step_eager_ms": step2_eager_ms,
            "steady_graph_weights_equal_eager": graph_equal,
            **({"steady_graph_error": graph_err} if graph_err else {}),
            "timing": "ms_per_step: mean over the 5 steps of BASELINE config 5 = (step 1 + 4 x "
                      "steady step) / 5; step 1 eager wave executor (142 GiB peak), steady step "
                      "one CUDA graph replay; every plaintext re-encoded, samples freshly "
                      "encrypted; wall clock, device sync on both sides",
            "steady_note": "step 1 runs on freshly encrypted top-level weights; steps 2..5 on "
                           "the refreshed weights at the refresh level: the recorded second "
                           "train_iteration (tests/golden/c5_trace.npz ops_step2)",
            "step2_weights_max_abs_err_vs_sim": float(err2[kind < 2].max()),
            "step2_velocities_max_abs_err_vs_sim": float(err2[kind >= 2].max()),
            "first_step_ms": 1e3 * times[0],
            "ops": len(prog.ops) - prog.n_setup, "waves": len(ex.waves),
            "bootstraps_per_step": int(sum(1 for o in prog.ops if o[0] == "bs")),
            "keygen_s": keygen_s, "max_group": max_group,
            "weights_max_abs_err_vs_sim": float(err[kind < 2].max()),
            "velocities_max_abs_err_vs_sim": float(err[kind >= 2].max()),
            "velocities_max_abs": float(mag[kind >= 2].max()),
            "peak_mem_gib": torch.cuda.max_memory_allocated() / 2**30,
            "workload": "64->64->64->64->64->2, batch 256, N=2^16, L=32 (16 user + 16 bootstrap "
                        "levels, insecure-test), P = 13 x 60 bits, real bootstrapping"}


if __name__ == "__main__":
    print(json.dumps(run(reps=int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                         max_group=int(sys.argv[2]) if len(sys.argv) > 2 else 64)))
