"""The fused peer-store exchange's plumbing on one device: a one-rank NCCL
group, torch symmetric memory for the receive buffer (symmetric_recv), the
scatter kernel storing into it, the symmetric-memory barrier, the unpack --
and bench.py's fused companion (setup agreement, byte-equality check against
the NCCL path, timing) on the same group.  With one rank nothing crosses
NVLink; this checks the API calls and the code path, not the fabric."""

import os
import socket
import sys
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        import bench
        import paper_1708_01873_b200 as br
        from paper_1708_01873_b200 import sharded

        b = 20
        x = torch.empty((1 << b) * 8, dtype=torch.uint8, device=dev).random_(0, 256).view(torch.complex64)
        try:
            peers, barrier, keep = sharded.symmetric_recv(x.numel(), x.dtype, dev)
        except Exception as exc:  # symmetric memory unavailable in this build
            q.put(("skip", f"{type(exc).__name__}: {exc}"[:300]))
            return
        out = sharded.sharded_bitrev_p2p(x, b, peers, 0, barrier)
        torch.cuda.synchronize()
        ok = torch.equal(out.view(torch.uint8), br.oracle_permute(x, b).view(torch.uint8))
        rec = bench.fused_p2p_companion(torch, dist, sharded, x, b, 0, 1, 3,
                                        torch.cuda.current_stream(dev))
        q.put(("ok", ok, rec))
    finally:
        dist.destroy_process_group()


def test_symmetric_memory_p2p_one_rank(cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    if res[0] == "skip":
        pytest.skip(res[1])
    _, ok, rec = res
    assert ok
    assert rec.get("value") and rec["value"] > 0, rec
    assert rec["checked"].startswith("byte-equal")
