"""Config-3 bootstrapping: CUDA-event time per stage (ModRaise, each CtS/StC
level, the two EvalMods) for a batch of 1 and of 4 ciphertexts, and the kernel
breakdown of the batch-4 call (the training steps' batched refresh)."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api, ring
from paper_2506_19693_b200 import bootstrap as BS
from paper_2506_19693_b200.backend import GpuCiphertext
from paper_2506_19693_b200.scheme import SchemeParams

n, L = 1 << 16, 24
params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,),
                      scale_bits=45, level=L, bootstrap_depth=16)
cust = he_api.keygen(params, set(), backend="ckks", rng_seed=11, prime_layout="bootstrap",
                     dnum=3, secret_hw=192, real_bootstrap=True)
be = cust.backend
rng = np.random.default_rng(3)
ct = be._encrypt_values(rng.uniform(-1, 1, n // 2), 0)
be.bootstrap_ct(ct)  # build the bootstrapper, keys, plaintext caches
rec = []


def timed(name, fn):
    def w(*a, **k):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = fn(*a, **k)
        e.record()
        rec.append((name, s, e))
        return r
    return w


B = BS.Bootstrapper
B._linear = timed("linear", B._linear)
if len(sys.argv) > 1 and sys.argv[1] == "evalmod":  # EvalMod internals instead
    for nm in ("_mul", "_add", "_add_const", "_double", "_drop_to", "_chebyshev_basis"):
        setattr(B, nm, timed(nm, getattr(B, nm)))
B._evalmod = timed("evalmod", B._evalmod)
be.mod_raise = timed("mod_raise", be.mod_raise)
for bsz in (1, 4):
    data = ct.data.unsqueeze(0).expand(bsz, -1, -1, -1).contiguous()
    for rep in range(2):
        rec.clear()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        be.bootstrap_batch(data, 0)
        torch.cuda.synchronize(); wall = 1e3 * (time.perf_counter() - t0)
    stages = [(nm, round(s.elapsed_time(e), 2)) for nm, s, e in rec]
    if len(sys.argv) > 1:
        agg = {}
        for nm, t in stages:
            a = agg.setdefault(nm, [0, 0.0]); a[0] += 1; a[1] = round(a[1] + t, 2)
        stages = agg
    print(json.dumps({"batch": bsz, "wall_ms": round(wall, 2), "stages": stages}))
ring.TIMER = ring.KernelTimer()
be.bootstrap_batch(ct.data.unsqueeze(0).expand(4, -1, -1, -1).contiguous(), 0)
summ = ring.TIMER.summary(); ring.TIMER = None
print(json.dumps({k: [round(d["ms"], 2), d["calls"]] for k, d in sorted(summ.items(), key=lambda x: -x[1]["ms"])}))
