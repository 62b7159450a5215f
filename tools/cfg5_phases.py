"""cfg5's local phases on one GPU (measurement tool, not product code).

For G = 2/4/8 (b = 32 complex64, shard b_local = 32 - log2 G) time, with CUDA
events over `reps` launches after warm-up, each local step of the sharded plan
on a shard-sized array:
  local   : bitrev_oop of the shard (the K = 1 pack)
  pack    : bitrev_sharded_pack with K = 4 exchange rounds (scatter kernel)
  scatter : bitrev_sharded_scatter into G local receive buffers (the fused p2p
            step, stores staying on this device)
  unpack  : bitrev_sharded_unpack of a full receive buffer
GB/s = 2 * shard bytes / time and the fraction of MEASURED_PEAKS hbm_gbs.
One JSON line per (G, phase).
"""

import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1708_01873_b200 import _core, sharded  # noqa: E402

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = torch.device("cuda", 0)
    b = 32
    for G in (2, 4, 8):
        g = G.bit_length() - 1
        bl = b - g
        n = 1 << bl
        x = torch.empty(n * 8, dtype=torch.uint8, device=dev).random_(0, 256).view(torch.complex64)
        y = torch.empty_like(x)
        S = n * 8
        recv = [torch.empty(n, dtype=torch.complex64, device=dev) for _ in range(G)]
        phases = {
            "local": lambda: _core.launch_oop(x, y, bl),
            "pack_k4": lambda: sharded._pack(x, bl, g, 2),
            "scatter": lambda: sharded._scatter(x, bl, g, 0, recv),
            "unpack": lambda: sharded._unpack(x, bl, g, y),
        }
        for name, fn in phases.items():
            t = timed(fn)
            gbs = 2 * S / t / 1e9
            print(json.dumps({"G": G, "b_local": bl, "phase": name, "ms": t * 1e3, "gbs": gbs,
                              "frac": gbs / PEAK, "shard_bytes": S}), flush=True)
        del x, y, recv
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
