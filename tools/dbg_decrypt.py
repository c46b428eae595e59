import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from oracle import ckks_oracle as O
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.scheme import SchemeParams
g = np.load("tests/golden/ref_ckks_n512.npz")
n, level, sb = (int(v) for v in g["params"])
params = SchemeParams(poly_degree=n, modulus_chain=tuple(int(v) for v in g["chain"]), scale_bits=sb, level=level)
cust = he_api.keygen(params, [1,3,-1], backend="ckks", rng_seed=11)
be = cust.backend
orc = O.OracleCkks(n, tuple(int(v) for v in g["chain"]), 40, level, rotation_steps=[], rng_seed=11)
ct = be.payload_from_planes(g["out_add"], level)
ph = be._phase(ct)
oct_ = O.ct_from_u64(g["out_add"], level, orc.chain)
oph = orc.phase(oct_)
print("phase equal:", np.array_equal(ph.cpu().numpy(), oph.to_u64()))
m = ph.shape[0]
f = be.chain.to_f64(ph, m)[0].cpu().numpy()
want = np.array([float(c) for c in O.lift_centered(oph, orc.chain)])
print("f64 max diff", np.max(np.abs(f - want)), f[:4], want[:4])
# small known values
vals = np.array([0, 1, -1, 5, -7, 2**40, -(2**40), 123456789012], dtype=np.int64)
x = np.zeros(n, dtype=np.int64); x[:len(vals)] = vals
r = be.chain.from_i64(torch.from_numpy(x).cuda(), m)[0]
print("small:", be.chain.to_f64(r, m)[0].cpu().numpy()[:len(vals)])
r2 = be.chain.from_i64(torch.from_numpy(x).cuda(), 3)[0]
print("small3:", be.chain.to_f64(r2, 3)[0].cpu().numpy()[:len(vals)])
