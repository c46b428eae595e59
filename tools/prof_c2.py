"""Profiling driver for ncu: one config-2 step (batch NTT/iNTT, HMult, HRot at
N=2^16, L=24, dnum=3, batch 64) between cudaProfilerStart/Stop, after keygen
and one warm-up step.  Run as `python tools/prof_c2.py [batch]`."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_19693_b200 import he_api  # noqa: E402

bsz = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = int(sys.argv[2]) if len(sys.argv) > 2 else 24
params, k = bench.c2_params(L)
rng = np.random.default_rng(1234)
steps = [int(s) for s in rng.integers(1, 1 << 15, bsz)]
cust = he_api.keygen(params, set(steps), backend="ckks", rng_seed=99, prime_layout="baseline",
                     dnum=bench.DNUM, secret_hw=192)
be = cust.backend
lvl = params.level
m = be.chain.level_limbs[lvl]
n = 1 << bench.N_LOG
g = torch.Generator(device="cuda")
g.manual_seed(7)
def rb():
    t = torch.empty(bsz, 2, m, n, dtype=torch.int64, device="cuda")
    for i, p in enumerate(be.chain.limbs_at(lvl)):
        t[:, :, i].random_(0, p, generator=g)
    return t.view(torch.uint64)
A, B = rb(), rb()
X = torch.empty_like(A)
def step():
    X.copy_(A)
    be.batch_ntt(X, lvl)
    be.batch_ntt(X, lvl, inverse=True)
    be.batch_hmult(A, B, lvl)
    be.batch_hrot(A, steps, lvl)
step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("prof_c2 ok")
