import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import make_params
path = "tests/golden/c1_trace.npz"; z = np.load(path); prog = Program.load(path)
n, level, sb = (int(v) for v in z["params"])
cust = he_api.keygen(make_params(level=level, scale_bits=sb, poly_degree=n), [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3, prime_layout="baseline", secret_hw=64)
env = prog.run(cust, 0, prog.n_setup)
ex = WaveExecutor(prog, cust)
be = cust.backend
orig = be._decrypt_values
marks = []
def wrapped(ct):
    marks.append(("dec_enter", time.perf_counter()))
    r = orig(ct)
    marks.append(("dec_exit", time.perf_counter()))
    return r
be._decrypt_values = wrapped
for rep in range(3):
    marks.clear()
    be._enc_cache.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e0.record()
    ex.run(dict(env), only_after_setup=True)
    t_ret = time.perf_counter()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"rep {rep}: wall {1e3*(t1-t0):.2f} ms, run() returned at {1e3*(t_ret-t0):.2f} ms; first decrypt entered at {1e3*(marks[0][1]-t0):.2f} ms, exited {1e3*(marks[1][1]-t0):.2f}; last dec exit {1e3*(marks[-1][1]-t0):.2f}")
