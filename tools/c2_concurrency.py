"""Config-2 HMult and HRot batches: sequential vs on two streams (experiment)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2506_19693_b200 import he_api
L, bsz = 24, 64
params, k = bench.c2_params(L)
rng = np.random.default_rng(1234)
steps = [int(s) for s in rng.integers(1, 1 << 15, bsz)]
cust = he_api.keygen(params, set(steps), backend="ckks", rng_seed=99, prime_layout="baseline",
                     dnum=bench.DNUM, secret_hw=192)
be = cust.backend
lvl = params.level
m = be.chain.level_limbs[lvl]
g = torch.Generator(device="cuda"); g.manual_seed(7)
def rb():
    t = torch.empty(bsz, 2, m, 1 << 16, dtype=torch.int64, device="cuda")
    for i, p in enumerate(be.chain.limbs_at(lvl)):
        t[:, :, i].random_(0, p, generator=g)
    return t.view(torch.uint64)
A, B = rb(), rb()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def seq():
    be.batch_hmult(A, B, lvl); be.batch_hrot(A, steps, lvl)
def conc():
    cur = torch.cuda.current_stream()
    sa.wait_stream(cur); sb.wait_stream(cur)
    with torch.cuda.stream(sa): be.batch_hmult(A, B, lvl)
    with torch.cuda.stream(sb): be.batch_hrot(A, steps, lvl)
    cur.wait_stream(sa); cur.wait_stream(sb)
for name, fn in (("seq", seq), ("conc", conc), ("seq", seq), ("conc", conc)):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 5, "ms")
