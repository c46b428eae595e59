"""Config 4 (SURVEY App. B substitution: 196->128->10, batch 128, N=2^16) with
real bootstrapping: the reference train_iteration's HE calls, wave-batched."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import SchemeParams


# training-step key switches over Q u P' with P' the first special primes above
# the widest digit of the level (backend.B200CkksCore low_special): levels <= 8 (digits <= 375 bits) over 7 x 60-bit special primes, levels 9..24
# (digits <= 480 bits) over 9;
# bootstrapping keeps the full P
LOW_SPECIAL = [(8, 7), (24, 9)]

def run(reps=2, verbose=True, graph=True, special=660):
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c4_trace.npz")
    z = np.load(path); prog = Program.load(path)
    n, L, sb, bd = (int(v) for v in z["params"])
    params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (special,),
                          scale_bits=45, level=L, bootstrap_depth=bd)
    t0 = time.perf_counter()
    cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=4,
                         prime_layout="bootstrap", dnum=3, secret_hw=192, real_bootstrap=True,
                         low_special=LOW_SPECIAL)
    torch.cuda.synchronize(); keygen_s = time.perf_counter() - t0
    env = prog.run(cust, 0, prog.n_setup)
    ex = WaveExecutor(prog, cust)
    times = []
    out = None
    for rep in range(reps):
        torch.cuda.reset_peak_memory_stats()
        cust.backend._enc_cache.clear()  # every step re-encodes its plaintexts
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = ex.run(dict(env), only_after_setup=True)
        torch.cuda.synchronize(); times.append(time.perf_counter() - t0)
        if verbose:
            print(f"step {rep}: {times[-1]*1e3:.1f} ms, peak mem {torch.cuda.max_memory_allocated()/2**30:.1f} GiB", flush=True)
    w = np.stack([cust.backend._decrypt_values(out[o]) for o in prog.outputs])
    graph_ms = None
    if graph:
        from paper_2506_19693_b200.graphs import GraphedStep

        gs = GraphedStep(ex, env, warmup=1)
        gt = []
        for rep in range(reps):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            og = gs.step()
            torch.cuda.synchronize(); gt.append(time.perf_counter() - t0)
        wg = np.stack([cust.backend._decrypt_values(og[o]) for o in prog.outputs])
        graph_ms = 1e3 * min(gt)
        from paper_2506_19693_b200.graphs import eager_equivalent
        oe = eager_equivalent(gs)
        graph_equal = bool(np.array_equal(wg, np.stack([cust.backend._decrypt_values(oe[o]) for o in prog.outputs])))
    err = np.max(np.abs(w - z["sim_weights"]), axis=1)  # layer w, classifier w, velocities
    mag = np.max(np.abs(z["sim_weights"]), axis=1)
    step1_ms = graph_ms if graph_ms is not None else 1e3 * min(times)
    # steady state: the trace's second train_iteration, on the weights and
    # velocities step 1 left (refreshed to the refresh level by its bootstraps)
    if graph:
        del gs, og
    prog2 = Program.load_step2(path)
    env2 = {k: out[k] for k in prog.keep}
    del out
    ex2 = WaveExecutor(prog2, cust)
    t2 = []
    for rep in range(reps):
        cust.backend._enc_cache.clear()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out2 = ex2.run(dict(env2), only_after_setup=True)
        torch.cuda.synchronize(); t2.append(time.perf_counter() - t0)
    w2 = np.stack([cust.backend._decrypt_values(out2[o]) for o in prog2.outputs])
    step2_ms = 1e3 * min(t2)
    step2_eager_ms = step2_ms
    if graph:
        del out2
        gs2 = GraphedStep(ex2, env2, warmup=1)
        g2 = []
        for rep in range(reps):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            og2 = gs2.step()
            torch.cuda.synchronize(); g2.append(time.perf_counter() - t0)
        wg2 = np.stack([cust.backend._decrypt_values(og2[o]) for o in prog2.outputs])
        oe2 = eager_equivalent(gs2)
        graph_equal = graph_equal and bool(np.array_equal(wg2, np.stack([cust.backend._decrypt_values(oe2[o]) for o in prog2.outputs])))
        step2_ms = 1e3 * min(g2)
    err2 = np.max(np.abs(w2 - z["sim_weights_step2"]), axis=1)
    res_graph = {} if graph_ms is None else {
        "ms_per_step_eager_waves": (1e3 * min(times) + 7 * step2_eager_ms) / 8,
        "graph_weights_equal_eager": graph_equal,
        "timing": "ms_per_step: mean over the 8 steps of BASELINE config 4 = (step 1 + 7 x "
                  "steady step) / 8; each step (4 real bootstraps included) one CUDA graph "
                  "replay, every plaintext re-encoded, samples freshly encrypted; wall clock, "
                  "device sync on both sides"}
    return {"ms_per_step": (step1_ms + 7 * step2_ms) / 8, **res_graph, "steps": 8,
            "step1_ms": step1_ms, "steady_step_ms": step2_ms,
            "steady_note": "step 1 runs on freshly encrypted top-level weights (levels 24..17, "
                           "the 60-bit bootstrap primes still present); steps 2..8 on the "
                           "refreshed weights at the refresh level (levels 8..1): the recorded "
                           "second train_iteration (tests/golden/c4_trace.npz ops_step2)",
            "step2_weights_max_abs_err_vs_sim": float(err2[:2].max()),
            "step2_velocities_max_abs_err_vs_sim": float(err2[2:].max()),
            "first_step_ms": 1e3 * times[0], "ops": len(prog.ops) - prog.n_setup,
            "waves": len(ex.waves), "bootstraps_per_step": 4, "keygen_s": keygen_s,
            "weights_max_abs_err_vs_sim": float(err[:2].max()),
            "velocities_max_abs_err_vs_sim": float(err[2:].max()),
            "velocities_max_abs": float(mag[2:].max()),
            "peak_mem_gib": torch.cuda.max_memory_allocated() / 2**30,
            "workload": "196->128->10, batch 128, N=2^16, L=24 (8 user + 16 bootstrap levels), real bootstrapping"}


if __name__ == "__main__":
    print(json.dumps(run(reps=int(sys.argv[1]) if len(sys.argv) > 1 else 2)))
