"""Experiment hook: CKB_L2_PERSIST_MB=<n> sets cudaLimitPersistingL2CacheSize before the
benchmark (does the evict_last policy of the NTT's first-phase stores need a carve-out?)."""
import ctypes
import os

import torch


def apply():
    mb = os.environ.get("CKB_L2_PERSIST_MB")
    if not mb:
        return
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    rt = None
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            rt = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if rt is None:
        import glob
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
        rt = ctypes.CDLL(cands[0])
    rc = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(int(mb) << 20))  # cudaLimitPersistingL2CacheSize
    val = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(val), 6)
    print(f"# persisting L2 limit: rc={rc} now {val.value >> 20} MiB", flush=True)
