"""Where does the config-1 step go: GPU kernel time (CUDA events per wrapper) vs wall."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api, ring
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import make_params
path = "tests/golden/c1_trace.npz"; z = np.load(path); prog = Program.load(path)
n, level, sb = (int(v) for v in z["params"])
cust = he_api.keygen(make_params(level=level, scale_bits=sb, poly_degree=n), [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3, prime_layout="baseline", secret_hw=64)
env = prog.run(cust, 0, prog.n_setup)
ex = WaveExecutor(prog, cust)
for rep in range(2):
    cust.backend._enc_cache.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter(); ex.run(dict(env), only_after_setup=True); torch.cuda.synchronize()
    print("wall ms", 1e3 * (time.perf_counter() - t0))
ring.TIMER = ring.KernelTimer()
torch.cuda.synchronize(); t0 = time.perf_counter(); ex.run(dict(env), only_after_setup=True); torch.cuda.synchronize()
wall = 1e3 * (time.perf_counter() - t0)
summ = ring.TIMER.summary(); ring.TIMER = None
tot = sum(d["ms"] for d in summ.values())
print("instrumented wall ms", wall, "sum of kernel ms", tot, "launches", sum(d["launches"] for d in summ.values()))
for k, d in sorted(summ.items(), key=lambda x: -x[1]["ms"]): print(f"  {k:18s} {d['ms']:8.2f} ms {d['calls']:5d} calls")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); ex.run(dict(env), only_after_setup=True); torch.cuda.synchronize(); pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(15)
