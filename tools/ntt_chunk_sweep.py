"""Sweep ckb_ring.ntt_chunk_bytes (rows per L2-resident chunk) on the N=2^16
NTT micro-benchmark: python tools/ntt_chunk_sweep.py [bits] [rows ...]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import _native as nat  # noqa: E402
from paper_2506_19693_b200.ring import U64  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 40
os.environ["NTT_BITS"] = str(bits)
sweep = [int(a) for a in sys.argv[2:]] or [74, 96, 111, 128, 148, 192, 222, 296]

# reuse ntt_micro's chain builder without running its benchmark
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ntt_micro.py")).read()
ns = {"__file__": os.path.join(os.path.dirname(os.path.abspath(__file__)), "ntt_micro.py")}
exec(src.split("res = {}")[0], ns)
logn, rows, limbs = 16, 3072, 24
ch = ns["chain_for"](logn, limbs, bits)
n = 1 << logn
x = torch.randint(0, 2 ** (bits - 1), (rows, n), dtype=torch.int64, device="cuda").view(U64)
out = {}
for cr in sweep:
    ch.ring.ntt_chunk_bytes = cr * n * 8
    for _ in range(2):
        ch.ntt_fwd(x, limbs); ch.ntt_inv(x, limbs)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    reps = 10
    e[0].record()
    for _ in range(reps): ch.ntt_fwd(x, limbs)
    e[1].record()
    for _ in range(reps): ch.ntt_inv(x, limbs)
    e[2].record(); torch.cuda.synchronize()
    out[cr] = (round(e[0].elapsed_time(e[1]) / reps, 4), round(e[1].elapsed_time(e[2]) / reps, 4))
print(json.dumps({"bits": bits, "rows_per_chunk -> (fwd_ms, inv_ms)": out}))
