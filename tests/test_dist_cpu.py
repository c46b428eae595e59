"""World-size-2 gloo tests of the multi-GPU host logic (dist.py): sharding,
the exact residue all-reduce (int64 sum + per-limb mod, as the GPU path does
with NCCL + ckb_reduce) and max-over-ranks timing."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

PRIMES = [1099511922689, 1099512004609, 1152921504606830593]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19693_b200 import dist as D

    rng = np.random.default_rng(100 + rank)
    n = 64
    x = np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in PRIMES])
    primes = torch.tensor(PRIMES, dtype=torch.int64).view(-1, 1)

    def reduce_mod(t):  # CPU stand-in for GpuChain.reduce (test only)
        return torch.remainder(t.view(torch.int64), primes).view(torch.uint64)

    got = D.allreduce_residues(torch.from_numpy(x.copy()), reduce_mod)
    m = D.max_over_ranks(float(rank + 1))
    out[rank] = (got.numpy().tolist(), m, list(D.shard(10, rank, world)))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_allreduce_residues_exact():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    want = None
    xs = []
    for rank in range(world):
        rng = np.random.default_rng(100 + rank)
        xs.append(np.stack([rng.integers(0, p, 64, dtype=np.uint64) for p in PRIMES]))
    want = [[(int(a) + int(b)) % p for a, b in zip(xs[0][i], xs[1][i])] for i, p in enumerate(PRIMES)]
    for rank in range(world):
        got, m, sh = out[rank]
        assert got == want
        assert m == 2.0
    assert out[0][2] == list(range(0, 5)) and out[1][2] == list(range(5, 10))


def test_shard_covers_all():
    from paper_2506_19693_b200.dist import shard

    for n in (0, 1, 7, 64):
        for w in (1, 2, 3, 8):
            items = [i for r in range(w) for i in shard(n, r, w)]
            assert items == list(range(n))
