"""NTT micro-benchmark: forward+inverse over `rows` limbs of N=2^logn (CUDA events)."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import _l2persist  # noqa: E402  (tools/ on sys.path when run as a script)
_l2persist.apply()
from oracle import ckks_oracle as O
from paper_2506_19693_b200 import _native as nat
from paper_2506_19693_b200.ring import GpuChain, U64

def chain_for(logn, nprimes, bits=40):
    n = 1 << logn
    used = set(); primes = []
    for _ in range(nprimes):
        p = O.largest_ntt_prime_below(bits, 2 * n, used); used.add(p); primes.append(p)
    ch = GpuChain.__new__(GpuChain)
    ch.n, ch.log_n, ch.device = n, logn, torch.device("cuda")
    ch.all_primes = primes; ch.primes = primes; ch.special_primes = []; ch.lq, ch.k = len(primes), 0
    mods, ntt, pair = nat.build_tables(logn, primes)
    ch._mods = torch.from_numpy(mods).cuda(); ch._ntt = torch.from_numpy(ntt.reshape(-1)).cuda(); ch._pair = torch.from_numpy(pair.reshape(-1)).cuda()
    ch.ring = nat.CkbRing(logn, len(primes), ch._mods.data_ptr(), ch._ntt.data_ptr(), ch._pair.data_ptr(), (nat.ctypes.c_uint64 * 2)(*nat.f64_mask(primes)))
    ch.ring_p = nat.ctypes.pointer(ch.ring); ch._maps = {}
    return ch

res = {}
BITS = int(os.environ.get("NTT_BITS", "40"))  # 60: the integer (Shoup) path
for logn, rows, limbs in [(16, 3072, 24), (12, 2304, 9)]:
  try:
      ch = chain_for(logn, limbs, BITS)
      n = 1 << logn

      x = torch.randint(0, 2**(BITS - 1), (rows, n), dtype=torch.int64, device="cuda").view(U64)
      ref = x.clone()
      for _ in range(3):
          ch.ntt_fwd(x, limbs); ch.ntt_inv(x, limbs)
      assert torch.equal(x.view(torch.int64), ref.view(torch.int64))
      e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
      reps = 10
      e[0].record()
      for _ in range(reps): ch.ntt_fwd(x, limbs)
      e[1].record()
      for _ in range(reps): ch.ntt_inv(x, limbs)
      e[2].record(); torch.cuda.synchronize()
      f = e[0].elapsed_time(e[1]) / reps; i = e[1].elapsed_time(e[2]) / reps
      gb = 2 * rows * n * 8 / 1e9
      res[f"N=2^{logn} rows={rows}"] = {"fwd_ms": f, "inv_ms": i, "fwd_GBps": gb / (f / 1e3), "inv_GBps": gb / (i / 1e3)}
  except Exception as exc:
    res[f"N=2^{logn}"] = {"error": repr(exc)[:80]}
print(json.dumps({"lib": os.environ.get("CKB_LIB", "default"), "bits": BITS, **res}))
