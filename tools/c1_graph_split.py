"""Config-1 graphed step: replay time vs the eager refreshes."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.graphs import GraphedStep
from paper_2506_19693_b200.scheme import make_params
path = "tests/golden/c1_trace.npz"; z = np.load(path); prog = Program.load(path)
n, level, sb = (int(v) for v in z["params"])
cust = he_api.keygen(make_params(level=level, scale_bits=sb, poly_degree=n), [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3, prime_layout="baseline", secret_hw=64)
env = prog.run(cust, 0, prog.n_setup)
ex = WaveExecutor(prog, cust)
gs = GraphedStep(ex, env)
for rep in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    gs.graph.replay(); torch.cuda.synchronize(); t1 = time.perf_counter()
    e = dict(gs.out_env); ex.deferred = list(gs.deferred); ex.finish_deferred(e); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"replay {1e3*(t1-t0):.2f} ms, refreshes {1e3*(t2-t1):.2f} ms")
