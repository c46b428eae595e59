"""Host-side issue cost of the config-1 step (cProfile, cumulative)."""
import cProfile, os, pstats, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import make_params
path = "tests/golden/c1_trace.npz"; z = np.load(path); prog = Program.load(path)
n, level, sb = (int(v) for v in z["params"])
cust = he_api.keygen(make_params(level=level, scale_bits=sb, poly_degree=n), [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3, prime_layout="baseline", secret_hw=64)
env = prog.run(cust, 0, prog.n_setup)
ex = WaveExecutor(prog, cust)
for _ in range(2):
    cust.backend._enc_cache.clear(); ex.run(dict(env), only_after_setup=True)
torch.cuda.synchronize()
cust.backend._enc_cache.clear()
pr = cProfile.Profile(); pr.enable(); ex.run(dict(env), only_after_setup=True); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
