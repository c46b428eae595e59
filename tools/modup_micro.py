"""ModUp micro-benchmark at config-2 shapes (64 ct, L=24, dnum=3, skip_own):
CUDA-event time of ckb_modup alone; honours CKB_LIB for A/B of builds."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2506_19693_b200 import he_api

L, B = 24, 64
params, k = bench.c2_params(L)
cust = he_api.keygen(params, [], backend="ckks", rng_seed=1, prime_layout="baseline", dnum=3)
be = cust.backend
ch = be.chain
m, n = L, be.n
d = torch.randint(0, 2**39, (B, m, n), dtype=torch.int64, device="cuda").view(torch.uint64)
tab = be._bconv(m)
for _ in range(3):
    ch.modup(d, m, be.alpha, tab, batch=B, skip_own=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    ch.modup(d, m, be.alpha, tab, batch=B, skip_own=True)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("CKB_LIB", "default"), "modup ms", round(e0.elapsed_time(e1) / reps, 3))
