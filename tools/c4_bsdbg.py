import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.replay import Program
from paper_2506_19693_b200.executor import WaveExecutor
from paper_2506_19693_b200.scheme import SchemeParams
from paper_2506_19693_b200.backend import GpuCiphertext
path = "tests/golden/c4_trace.npz"
z = np.load(path); prog = Program.load(path)
n, L, sb, bd = (int(v) for v in z["params"])
params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,), scale_bits=45, level=L, bootstrap_depth=bd)
cust = he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=4, prime_layout="bootstrap", dnum=3, secret_hw=192, real_bootstrap=True)
be = cust.backend
orig = be.bootstrap_ct
def hooked(ct):
    before = be._decrypt_values(ct)
    lvl0 = GpuCiphertext(be._adjust_data(ct.data, ct.level, 0), 0) if ct.level else ct
    b0 = be._decrypt_values(lvl0)
    out = orig(ct)
    after = be._decrypt_values(out)
    print(f"bs: in level {ct.level} |v|max {np.max(np.abs(before)):.3e} adjust err {np.max(np.abs(b0-before)):.3e} bs err {np.max(np.abs(after-before)):.3e}", flush=True)
    return out
be.bootstrap_ct = hooked
env = prog.run(cust, 0, prog.n_setup)
out = WaveExecutor(prog, cust).run(dict(env), only_after_setup=True)
w = np.stack([be._decrypt_values(out[o]) for o in prog.outputs])
print("err per output", np.max(np.abs(w - z["sim_weights"]), axis=1), "max |w|", np.max(np.abs(z["sim_weights"]), axis=1))
