"""Packed residue transfer format (ckb_pack / ckb_unpack, backend.pack_batch):
the byte layout matches a numpy restatement of the format (w_l = 5 / 6 / 8
bytes per residue by prime size class, little-endian, an item's limbs back to
back), and unpack(pack(x)) == x on chains with 40-, 45- and 60-bit primes."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2506_19693_b200 import he_api  # noqa: E402
from paper_2506_19693_b200.scheme import SchemeParams, make_params  # noqa: E402


def _np_pack(x: np.ndarray, primes) -> bytes:
    """[items][limbs][N] uint64 -> the packed bytes (the format's definition)."""
    ws = [8 if p >= 1 << 48 else 6 if p >= 1 << 40 else 5 for p in primes]
    out = bytearray()
    for item in x:
        for row, w in zip(item, ws):
            b = row.astype("<u8").view(np.uint8).reshape(-1, 8)[:, :w]
            out += b.tobytes()
    return bytes(out)


@pytest.mark.parametrize("layout", ["c2", "boot"])
def test_pack_roundtrip_and_format(layout):
    n = 4096
    if layout == "c2":
        params = make_params(level=11, scale_bits=40, poly_degree=n, first_bits=40,
                             special_bits=120)
        opts = dict(prime_layout="baseline", dnum=3, secret_hw=64)
    else:
        params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 4 + (60,) * 2 + (360,),
                              scale_bits=45, level=6, bootstrap_depth=2)
        opts = dict(prime_layout="bootstrap", dnum=3, secret_hw=64)
    cust = he_api.keygen(params, set(), backend="ckks", rng_seed=3, **opts)
    be = cust.backend
    ch = be.chain
    rng = np.random.default_rng(5)
    lvl = params.level
    primes = ch.limbs_at(lvl)
    x = np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
                  for _ in range(6)]).reshape(3, 2, len(primes), n)
    d = torch.from_numpy(x).cuda()
    packed = be.pack_batch(d, lvl)
    assert packed.shape[0] == 3
    assert packed.cpu().numpy().tobytes() == _np_pack(x.reshape(6, len(primes), n), primes)
    back = be.unpack_batch(packed, lvl)
    assert torch.equal(back.view(torch.int64), d.view(torch.int64))
    # all limbs, special primes included (8-byte class)
    allp = ch.all_primes
    y = np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in allp])[None]
    ty = torch.from_numpy(y).cuda()
    pk = ch.pack(ty, 1, len(allp), ch.all_map())
    assert pk.cpu().numpy().tobytes() == _np_pack(y, allp)
    assert torch.equal(ch.unpack(pk, 1, len(allp), ch.all_map()).view(torch.int64),
                       ty.view(torch.int64))
