"""Config-4 step (argv[1] == "2": the steady second step): histogram of the wave executor's batched groups (kind, level,
batch size) and the kernel-time breakdown with rows per kernel."""
import collections, json, os, sys, time
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
if len(sys.argv) > 1 and sys.argv[1] == "2":
    out = ex.run(dict(env), only_after_setup=True)
    prog = Program.load_step2(path)
    env = {k: out[k] for k in Program.load(path).keep}
    del out
    ex = WaveExecutor(prog, cust)
hist = collections.Counter()
orig = WaveExecutor._run_group
def rec(self, key, idx, env_, pvals):
    k = key[0] if key[0] in ("rot", "enc") or key[0].startswith("bs") else key[0]
    lvl = key[1] if len(key) > 1 and isinstance(key[1], int) else -1
    hist[(k, lvl, len(idx))] += 1
    return orig(self, key, idx, env_, pvals)
WaveExecutor._run_group = rec
ex.run(dict(env), only_after_setup=True)
WaveExecutor._run_group = orig
rows = sorted(hist.items(), key=lambda kv: -kv[1] * kv[0][2])
print("groups (kind, level, batch): count")
for (k, lvl, b), c in rows[:40]:
    print(f"  {k:8s} L{lvl:<3d} B={b:<4d} x{c}")
ring.TIMER = ring.KernelTimer()
cust.backend._enc_cache.clear()
ex.run(dict(env), only_after_setup=True)
summ = ring.TIMER.summary(); ring.TIMER = None
for k, d in sorted(summ.items(), key=lambda x: -x[1]["ms"]):
    print(f"{k:18s} {d['ms']:8.1f} ms calls {d['calls']:6d} launches {d['launches']:6d} GB {d['bytes']/1e9:8.1f}  GB/s {d['bytes']/1e6/max(d['ms'],1e-9):7.0f}")
