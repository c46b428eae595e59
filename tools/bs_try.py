"""Bootstrapping trial: N=2^logn, L=24 x 45-bit, dnum=3, HW-192 secret."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.scheme import SchemeParams
from paper_2506_19693_b200.bootstrap import Bootstrapper, bootstrap_rotations

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 13
n = 1 << logn
L = 24
params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,), scale_bits=45,
                      level=L, bootstrap_depth=16)
t0 = time.time()
rots = bootstrap_rotations(params)
cust = he_api.keygen(params, rots, backend="ckks", rng_seed=1, prime_layout="bootstrap",
                     dnum=3, secret_hw=192, conjugation_key=True)
be = cust.backend
torch.cuda.synchronize()
print("keygen", time.time() - t0, "rots", len(rots), "alpha", be.alpha, "k", be.chain.k, flush=True)
print("scales", [round(np.log2(s), 4) for s in be.chain.scale_at[:3]], "...", round(np.log2(be.chain.scale_at[-1]), 4))
bs = Bootstrapper(be)
rng = np.random.default_rng(0)
v = rng.uniform(-1, 1, n // 2)
ct = be._encrypt_values(v, 0)
print("input err", np.max(np.abs(be._decrypt_values(ct) - v)))
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    out = bs.bootstrap(ct)
    torch.cuda.synchronize(); dt = time.time() - t0
    got = be._decrypt_values(out)
    err = np.max(np.abs(got - v))
    print(f"bootstrap {dt*1e3:.1f} ms level {out.level} max err {err:.3e} (2^{np.log2(err):.1f})", flush=True)
