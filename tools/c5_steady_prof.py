"""Config-5 steady step (the recorded second train_iteration): wall time vs
summed CUDA-event kernel time, and whether a CUDA graph of the step fits."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api, ring
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import SchemeParams

path = "tests/golden/c5_trace.npz"
z = np.load(path); prog = Program.load(path)
n, L, sb, bd = (int(v) for v in z["params"])
params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * (L - bd) + (60,) * bd + (780,),
                      scale_bits=45, level=L, bootstrap_depth=bd)
cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=5,
                     prime_layout="bootstrap", dnum=3, secret_hw=192, real_bootstrap=True)
env = prog.run(cust, 0, prog.n_setup)
mg = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ex = WaveExecutor(prog, cust, max_group=mg)
out = ex.run(dict(env), only_after_setup=True)
prog2 = Program.load_step2(path)
env2 = {k: out[k] for k in prog.keep}
del out, ex
torch.cuda.empty_cache()
ex2 = WaveExecutor(prog2, cust, max_group=mg)
for rep in range(2):
    torch.cuda.reset_peak_memory_stats()
    cust.backend._enc_cache.clear()
    if rep == 1:
        ring.TIMER = ring.KernelTimer()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    o2 = ex2.run(dict(env2), only_after_setup=True)
    torch.cuda.synchronize(); wall = 1e3 * (time.perf_counter() - t0)
    del o2
summ = ring.TIMER.summary(); ring.TIMER = None
print(json.dumps({"max_group": mg, "wall_ms": wall, "kernel_ms": sum(d["ms"] for d in summ.values()),
                  "peak_gib": torch.cuda.max_memory_allocated() / 2**30,
                  "kernels": {k: round(d["ms"], 1) for k, d in sorted(summ.items(), key=lambda x: -x[1]["ms"])}}))
