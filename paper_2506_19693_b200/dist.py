"""Multi-GPU plumbing: one process per GPU over
torch.distributed (NCCL on GPUs, gloo in the CPU tests).

* ``shard(n, rank, world)`` — contiguous split of n independent items
  (ciphertexts of a batch, samples of a mini-batch).
* ``allreduce_residues(x, reduce_mod)`` — exact sum of RNS residue tensors
  across ranks: an int64 all-reduce (residues < 2^60, so up to 16 ranks cannot
  overflow 2^64) followed by a per-limb ``mod p`` (``GpuChain.reduce`` on the
  device).  This is the one exchange the ReBoot training step needs: the
  per-rank partial δW sums (nn.py:374-381) before the replicated update.
* ``max_over_ranks(ms)`` — timing is the max over ranks (bench contract).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

MAX_EXACT_RANKS = 16


def world() -> tuple:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(n: int, rank: int, world_size: int) -> range:
    base, extra = divmod(n, world_size)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def allreduce_residues(x: torch.Tensor, reduce_mod, group=None) -> torch.Tensor:
    """Sum uint64 residue tensors across ranks, exactly, then reduce mod p."""
    _, ws = world()
    if ws > MAX_EXACT_RANKS:
        raise ValueError(f"exact residue all-reduce supports <= {MAX_EXACT_RANKS} ranks")
    if ws > 1:
        y = x.view(torch.int64)
        staged = y.is_cuda and dist.get_backend(group) == "gloo"
        y = y.cpu() if staged else y.clone()  # NCCL reduces in place on the device
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
        x = (y.to(x.device) if staged else y).view(torch.uint64)
    return reduce_mod(x)


def reduce_scalar(value, op=None, dtype=torch.float64):
    """All-reduce one number (default MAX); gloo groups reduce it on the host,
    NCCL groups on the current device."""
    _, ws = world()
    if ws == 1:
        return value
    dev = "cpu" if dist.get_backend() == "gloo" else torch.device("cuda",
                                                                 torch.cuda.current_device())
    t = torch.tensor([value], dtype=dtype, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op is None else op)
    return t.item()


def max_over_ranks(value: float, device=None) -> float:
    return float(reduce_scalar(float(value)))
