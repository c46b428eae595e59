"""Variance of the config-2 HMult+HRot pair on two streams (the bench's value):
per-iteration CUDA-event times over many repetitions, host enqueue time beside
them.  python tools/pair_var.py [reps]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_19693_b200 import he_api  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
L, bsz = 24, 64
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
prio = os.environ.get("PAIR_PRIO", "")  # "hm" / "hr": that stream at high priority
s1 = torch.cuda.Stream(priority=-1 if prio == "hm" else 0)
s2 = torch.cuda.Stream(priority=-1 if prio == "hr" else 0)


def pair():
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


for _ in range(3):
    pair()
torch.cuda.synchronize()
res = []
for mode in ("back_to_back", "synced"):
    ts, hs = [], []
    evs = []
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode == "synced":
            torch.cuda.synchronize()
        h0 = time.perf_counter()
        a.record()
        pair()
        b.record()
        hs.append(1e3 * (time.perf_counter() - h0))
        evs.append((a, b))
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in evs]
    res.append({"mode": mode, "pair_ms": [round(t, 2) for t in ts],
                "host_enqueue_ms": [round(h, 2) for h in hs],
                "mean": round(float(np.mean(ts)), 3), "median": round(float(np.median(ts)), 3)})
print(json.dumps(res))
