"""The top-bit sharded plan on CPU.

1. A numpy simulation of the three steps (local reversal of b-g bits, equal
   chunk all-to-all, [G x C] -> [C x G] interleave with rev_g on rows) equals
   the oracle for many (b, G).
2. The product's exchange, paper_1708_01873_b200.sharded.sharded_bitrev, runs
   under torch.distributed with the gloo backend at world sizes 2 and 4: its
   own all_to_all_single rounds move the data; only the two local CUDA steps
   (pack, unpack) are injected as oracle-backed CPU callables (the kernels
   behind them are covered by the GPU tests).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1708_01873_b200 import sharded


def unpack_np(recv, b_local, g):
    G = 1 << g
    C = 1 << (b_local - g)
    out = np.empty_like(recv)
    for r in range(G):
        out[orc.rev_naive(r, g)::G] = recv[r * C:(r + 1) * C]
    return out


def simulate(x, b, G):
    g = G.bit_length() - 1
    bl = b - g
    S, C = 1 << bl, 1 << (bl - g)
    staged = [orc.oracle_permute(x[r * S:(r + 1) * S], bl) for r in range(G)]
    outs = []
    for d in range(G):
        recv = np.concatenate([staged[r][d * C:(d + 1) * C] for r in range(G)])
        outs.append(unpack_np(recv, bl, g))
    return np.concatenate(outs)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("b", [6, 7, 9, 12, 16])
def test_plan_simulation_matches_oracle(b, G):
    if 2 * (G.bit_length() - 1) > b:
        pytest.skip("plan needs b >= 2g")
    x = np.random.default_rng(b * 10 + G).integers(0, 1 << 60, 1 << b, dtype=np.int64)
    assert np.array_equal(simulate(x, b, G), orc.oracle_permute(x, b))


def test_plan_rejects_too_many_ranks():
    with pytest.raises(ValueError, match="b >= 2"):
        sharded.check_plan(3, 4)
    with pytest.raises(ValueError, match="power of two"):
        sharded.check_plan(10, 3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def pack_np(shard, b_local, g, kb):
    """Step 1 as the pack kernel lays it out: [sub-chunk c][destination d][k']."""
    G, K = 1 << g, 1 << kb
    S = 1 << (b_local - g - kb)
    L = orc.oracle_permute(shard, b_local)           # L[d*C + c*S + k']
    return np.ascontiguousarray(L.reshape(G, K, S).transpose(1, 0, 2)).reshape(-1)


def test_pack_layout_is_plain_reversal_for_one_chunk():
    x = np.arange(1 << 10, dtype=np.int64)
    assert np.array_equal(pack_np(x, 10, 2, 0), orc.oracle_permute(x, 10))


def _worker(rank, world, port, b, q, chunks=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        bl = b - g
        full = np.random.default_rng(b).integers(0, 1 << 60, 1 << b, dtype=np.int64)
        local = torch.from_numpy(full[rank << bl:(rank + 1) << bl].copy())

        # only the two local CUDA steps are replaced; the exchange is the
        # product's own all_to_all_single rounds (gloo implements them)
        def pack(t, bits, gg, kb):
            return torch.from_numpy(pack_np(t.numpy(), bits, gg, kb))

        def unpack(recv, bits, gg, out):
            out.copy_(torch.from_numpy(unpack_np(recv.numpy(), bits, gg)))

        out = sharded.sharded_bitrev(local, b, chunks=chunks, pack=pack, unpack=unpack)
        expect = orc.oracle_permute(full, b)[rank << bl:(rank + 1) << bl]
        q.put((rank, bool(np.array_equal(out.numpy(), expect))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks,b", [(2, 1, 10), (4, 1, 10), (2, 4, 14), (4, 2, 14),
                                            (4, 4, 16), (2, 4, 8)])
def test_sharded_bitrev_gloo(world, chunks, b):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, b, q, chunks))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {r: True for r in range(world)}


def test_sharded_bitrev_rejects_host_shards():
    """No CPU path: the default local steps need a CUDA shard."""
    with pytest.raises(ValueError, match="CUDA"):
        sharded.sharded_bitrev(torch.zeros(1 << 10, dtype=torch.int64), 10)
