"""The sharded plan end to end with its real kernels on one device: two ranks
(processes) on cuda:0 over gloo run sharded_bitrev on their shards -- the
CUDA pack, the product's all_to_all_single rounds (gloo moves the bytes
through host memory; on a node it is NCCL over NVLink), the CUDA unpack -- and
the concatenated shards must equal the oracle byte for byte.  The ranks'
kernels never wait on each other; this is a functional test, not a timing.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, b, chunks, dtype_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1708_01873_b200 import sharded

        dtype = getattr(torch, dtype_name)
        g = world.bit_length() - 1
        E = torch.empty(0, dtype=dtype).element_size()
        full = np.random.default_rng(b).integers(0, 256, (1 << b) * E, dtype=np.uint8)
        S = 1 << (b - g)
        local = torch.from_numpy(full[rank * S * E:(rank + 1) * S * E].copy()).to("cuda:0").view(dtype)
        try:
            out = sharded.sharded_bitrev(local, b, chunks=chunks)
        except RuntimeError as exc:  # a gloo build without CUDA all-to-all
            q.put((rank, "skip: " + str(exc)[:200]))
            return
        torch.cuda.synchronize()
        q.put((rank, out.view(torch.uint8).cpu().numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks,b,dtype", [(2, 1, 20, "complex64"), (2, 4, 20, "float32"),
                                                  (4, 2, 18, "complex128")])
def test_sharded_bitrev_two_processes_one_device(cuda, world, chunks, b, dtype):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, b, chunks, dtype, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    if any(isinstance(v, str) for v in res.values()):
        pytest.skip(next(v for v in res.values() if isinstance(v, str)))
    E = torch.empty(0, dtype=getattr(torch, dtype)).element_size()
    full = np.random.default_rng(b).integers(0, 256, (1 << b) * E, dtype=np.uint8)
    from oracle import oracle as orc

    words = full.view(np.uint64 if E >= 8 else np.uint32).reshape(1 << b, -1)
    want = orc.oracle_permute(words.T, b).T.reshape(-1).view(np.uint8)
    got = np.frombuffer(b"".join(res[r] for r in range(world)), dtype=np.uint8)
    assert np.array_equal(got, want)
