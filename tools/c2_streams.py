"""Stream-schedule experiment for the config-2 HMult + HRot pair (64 ct each):
how the two independent batches are split over CUDA streams.  Prints the
CUDA-event time of each schedule (mean of 5 after warm-up)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2506_19693_b200 import he_api  # noqa: E402

L, bsz = 24, 64
params, k = bench.c2_params(L)
rng = np.random.default_rng(1234)
steps = [int(s) for s in rng.integers(1, 1 << 15, bsz)]
cust = he_api.keygen(params, set(steps), backend="ckks", rng_seed=99, prime_layout="baseline",
                     dnum=3, secret_hw=192)
be = cust.backend
lvl = params.level
m, n = be.chain.level_limbs[lvl], 1 << 16
g = torch.Generator(device="cuda")
g.manual_seed(7)


def rb():
    t = torch.empty(bsz, 2, m, n, dtype=torch.int64, device="cuda")
    for i, p in enumerate(be.chain.limbs_at(lvl)):
        t[:, :, i].random_(0, p, generator=g)
    return t.view(torch.uint64)


A, B = rb(), rb()
streams = [torch.cuda.Stream() for _ in range(4)]


def run(plan, chunk):
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    prev = be.chain.set_ntt_chunk_bytes(chunk)
    for si, jobs in enumerate(plan):
        with torch.cuda.stream(streams[si]):
            for kind, lo, hi in jobs:
                if kind == "m":
                    be.batch_hmult(A[lo:hi], B[lo:hi], lvl)
                else:
                    be.batch_hrot(A[lo:hi], steps[lo:hi], lvl)
    be.chain.set_ntt_chunk_bytes(prev)
    for s in streams:
        cur.wait_stream(s)


plans = {
    "seq_1stream_96MB": ([[("m", 0, 64), ("r", 0, 64)]], 96 << 20),
    "pair_2streams_48MB": ([[("m", 0, 64)], [("r", 0, 64)]], 48 << 20),
    "pair_2streams_96MB": ([[("m", 0, 64)], [("r", 0, 64)]], 96 << 20),
    "pair_2streams_32MB": ([[("m", 0, 64)], [("r", 0, 64)]], 32 << 20),
    "pair_2streams_40MB": ([[("m", 0, 64)], [("r", 0, 64)]], 40 << 20),
    "pair_2streams_56MB": ([[("m", 0, 64)], [("r", 0, 64)]], 56 << 20),
    "pair_2streams_64MB": ([[("m", 0, 64)], [("r", 0, 64)]], 64 << 20),
    "pair_2streams_80MB": ([[("m", 0, 64)], [("r", 0, 64)]], 80 << 20),
    "halves_4streams_24MB": ([[("m", 0, 32)], [("m", 32, 64)], [("r", 0, 32)], [("r", 32, 64)]],
                             24 << 20),
    "offset_2streams_48MB": ([[("m", 0, 32), ("r", 0, 32)], [("r", 32, 64), ("m", 32, 64)]],
                             48 << 20),
    "offset_2streams_quarters": ([[("m", 0, 16), ("r", 0, 16), ("m", 16, 32), ("r", 16, 32),
                                   ("m", 32, 48), ("r", 32, 48), ("m", 48, 64), ("r", 48, 64)],
                                  [("r", 48, 64), ("m", 48, 64), ("r", 32, 48), ("m", 32, 48),
                                   ("r", 16, 32), ("m", 16, 32), ("r", 0, 16), ("m", 0, 16)]],
                                 48 << 20),
}
for name, (plan, chunk) in plans.items():
    for _ in range(2):
        run(plan, chunk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run(plan, chunk)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) / 5:8.3f} ms", flush=True)
