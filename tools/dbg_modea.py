import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200.scheme import SchemeParams
g = np.load("tests/golden/ref_ckks_n512.npz")
n, level, sb = (int(v) for v in g["params"])
params = SchemeParams(poly_degree=n, modulus_chain=tuple(int(v) for v in g["chain"]), scale_bits=sb, level=level)
cust = he_api.keygen(params, [1,3,-1], backend="ckks", rng_seed=11)
be = cust.backend
p1 = be.payload_from_planes(g["ct1"], level)
back = be.planes_of(p1)
print("roundtrip", np.array_equal(back, g["ct1"]))
x = torch.from_numpy(g["ct1"].astype(np.uint64)).cuda()
y = be.chain.ntt_fwd(x.clone(), 8)
z = be.chain.ntt_inv(y.clone(), 8)
print("rt2", torch.equal(z.view(torch.int64), x.view(torch.int64)))
print("shapes", x.shape, x.is_contiguous())
# per row check
for r in range(2):
    for l in range(8):
        a = x[r, l].clone(); b = be.chain.ntt_inv(be.chain.ntt_fwd(a.clone(), 1, be.chain.cmap((l,))), 1, be.chain.cmap((l,)))
        if not torch.equal(a.view(torch.int64), b.view(torch.int64)): print("row bad", r, l)
