"""Config-4 step breakdown: CUDA-event time per kernel wrapper (ring.KernelTimer),
split into the training ops and the 4 real bootstraps."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api, ring
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import SchemeParams

path = "tests/golden/c4_trace.npz"
z = np.load(path); prog = Program.load(path)
n, L, sb, bd = (int(v) for v in z["params"])
params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,),
                      scale_bits=45, level=L, bootstrap_depth=bd)
cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=4,
                     prime_layout="bootstrap", dnum=3, secret_hw=192, real_bootstrap=True)
env = prog.run(cust, 0, prog.n_setup)
ex = WaveExecutor(prog, cust)
ex.run(dict(env), only_after_setup=True)
be = cust.backend
# bootstrap alone
ct = env[next(iter(env))]
x = getattr(ct, "payload", ct)
torch.cuda.synchronize(); t0 = time.perf_counter(); be.bootstrap_ct(x); torch.cuda.synchronize()
print("one bootstrap ms", 1e3 * (time.perf_counter() - t0))
ring.TIMER = ring.KernelTimer()
be.bootstrap_ct(x)
bs = ring.TIMER.summary(); ring.TIMER = None
print("bootstrap kernels", json.dumps({k: [round(d["ms"], 2), round(d["f64_bytes"] / max(d["bytes"], 1), 2)] for k, d in sorted(bs.items(), key=lambda x: -x[1]["ms"])}))
ring.TIMER = ring.KernelTimer()
cust.backend._enc_cache.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
ex.run(dict(env), only_after_setup=True)
torch.cuda.synchronize(); wall = 1e3 * (time.perf_counter() - t0)
summ = ring.TIMER.summary(); ring.TIMER = None
tot = sum(d["ms"] for d in summ.values())
print(json.dumps({"wall_ms": wall, "kernel_ms": tot, "launches": sum(d["launches"] for d in summ.values()),
                  "kernels": {k: [round(d["ms"], 1), round(d["f64_bytes"] / max(d["bytes"], 1), 2)] for k, d in sorted(summ.items(), key=lambda x: -x[1]["ms"])}}))
