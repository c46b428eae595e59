"""Per-kernel CUDA-event times of one config-2 HMult batch + HRot batch (N=2^16,
L=24, dnum=3, k=6, 64 ct, sequential issue; ring.KernelTimer around every
wrapper) for A/B of builds: CKB_LIB=<variant .so> python tools/ks_micro.py [L] [B]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _l2persist  # noqa: E402  (tools/ on sys.path when run as a script)
_l2persist.apply()
import bench  # noqa: E402
from paper_2506_19693_b200 import he_api, ring  # noqa: E402

if os.environ.get("CKB_FUSE_KS"):  # A/B: 1 = fused digits NTT + inner product
    ring.GpuChain.fuse_ks_mac = os.environ["CKB_FUSE_KS"] == "1"

L = int(sys.argv[1]) if len(sys.argv) > 1 else 24
bsz = int(sys.argv[2]) if len(sys.argv) > 2 else 64
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
if os.environ.get("CKB_NTT_SPLIT") == "1":  # class-split NTT launches (ckb_ring flag)
    from paper_2506_19693_b200 import _native as _nat

    be.chain.set_ring_flag(_nat.RING_NTT_SPLIT, True)
if os.environ.get("CKB_LAZY") == "0":  # canonical basis-conversion outputs (A/B)
    from paper_2506_19693_b200 import _native as _nat0

    be.chain.set_ring_flag(_nat0.RING_LAZY_BCONV, False)
if os.environ.get("CKB_CHUNK_MB"):  # L2 budget of the sequential transforms
    be.chain.set_ntt_chunk_bytes(int(os.environ["CKB_CHUNK_MB"]) << 20)
X = torch.empty_like(A)
for _ in range(2):
    be.batch_hmult(A, B, lvl)
    be.batch_hrot(A, steps, lvl)
torch.cuda.synchronize()
reps = 5
res = {}
def ntt_stage():
    X.copy_(A)
    be.batch_ntt(X, lvl)
    be.batch_ntt(X, lvl, inverse=True)


for name, fn in (("hmult", lambda: be.batch_hmult(A, B, lvl)),
                 ("hrot", lambda: be.batch_hrot(A, steps, lvl)), ("ntt_stage", ntt_stage)):
    t = ring.KernelTimer()
    ring.TIMER = t
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ring.TIMER = None
    res[name] = {"total": round(e0.elapsed_time(e1) / reps, 3),
                 **{kk: round(v["ms"] / reps, 3) for kk, v in t.summary().items()}}
# the pair on two streams, untimed per kernel
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    prev = be.chain.set_ntt_chunk_bytes(48 << 20)
    with torch.cuda.stream(s1):
        be.batch_hmult(A, B, lvl)
    with torch.cuda.stream(s2):
        be.batch_hrot(A, steps, lvl)
    be.chain.set_ntt_chunk_bytes(prev)
    cur.wait_stream(s1)
    cur.wait_stream(s2)
e1.record()
torch.cuda.synchronize()
res["pair_ms"] = round(e0.elapsed_time(e1) / reps, 3)
tag = (os.environ.get("CKB_LIB") or "x/default/x").split("/")[-2]
if os.environ.get("CKB_CHUNK_MB"):
    tag += f"+chunk{os.environ['CKB_CHUNK_MB']}"
if os.environ.get("CKB_NTT_SPLIT") == "1":
    tag += "+split"
if os.environ.get("CKB_FUSE_KS") == "1":
    tag += "+fused"
if os.environ.get("CKB_LAZY") == "0":
    tag += "+eager_bconv"
print(tag, json.dumps(res))
