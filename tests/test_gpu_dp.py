"""Data-parallel training step on the GPU (dp.DataParallelExecutor,
SURVEY.md §8(e)): two ranks, each owning half of the c1 mini-batch, exchange
their partial δW sums with one exact residue all-reduce; the refreshed weights
must equal the single-process WaveExecutor's bit for bit.

The round's GPU budget is one B200, so both ranks run on cuda:0 and exchange
over gloo (host memory): no kernel of one rank waits on the other's, only the
all-reduce joins them.  On a multi-GPU node the same code runs one rank per
GPU over NCCL (bench.py --gpus N, c1_dp line)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _custodian(z):
    from paper_2506_19693_b200 import he_api
    from paper_2506_19693_b200.scheme import make_params

    n, level, sb = (int(v) for v in z["params"])
    params = make_params(level=level, scale_bits=sb, poly_degree=n)
    return he_api.keygen(params, [int(r) for r in z["rotations"]], backend="ckks", rng_seed=3,
                         prime_layout="baseline", secret_hw=64)


def _worker(rank, world, port, path, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19693_b200.dp import DataParallelExecutor
    from paper_2506_19693_b200.replay import Program

    prog, z = Program.load(path), np.load(path)
    cust = _custodian(z)
    ex = DataParallelExecutor(prog, cust, encs_per_sample=3)
    env = ex.run()
    planes = np.stack([cust.backend.planes_of(env[o]) for o in prog.outputs])
    np.save(os.path.join(outdir, f"rank{rank}.npy"), planes)
    np.save(os.path.join(outdir, f"bytes{rank}.npy"), np.array([ex.exchanged_bytes]))
    dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_dp_two_ranks_bit_identical_to_one(golden_dir):
    from paper_2506_19693_b200.executor import WaveExecutor
    from paper_2506_19693_b200.replay import Program

    path = os.path.join(golden_dir, "c1_trace.npz")
    prog, z = Program.load(path), np.load(path)
    cust = _custodian(z)
    env = WaveExecutor(prog, cust).run()
    want = np.stack([cust.backend.planes_of(env[o]) for o in prog.outputs])
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), path, d), nprocs=2, join=True)
        for r in range(2):
            got = np.load(os.path.join(d, f"rank{r}.npy"))
            assert np.array_equal(got, want), f"rank {r} differs"
            assert int(np.load(os.path.join(d, f"bytes{r}.npy"))[0]) > 0
