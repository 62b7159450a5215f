"""cfg5 unpack (bitrev_sharded_unpack) at the shard sizes of G = 2 / 4 / 8,
median of 10 event-timed launches; the grid's CTAs per SM come from
BITREV_B200_UNPACK_PER_SM (read once per process).  Measurement probe only."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import sharded  # noqa: E402

PEAK = 6551.7
per_sm = os.environ.get("BITREV_B200_UNPACK_PER_SM", "8")
dev = torch.device("cuda", 0)
for G in (2, 4, 8):
    g = G.bit_length() - 1
    bl = 32 - g
    n = 1 << bl
    x = torch.empty(n * 8, dtype=torch.uint8, device=dev).random_(0, 256).view(torch.complex64)
    y = torch.empty_like(x)
    for _ in range(3):
        sharded._unpack(x, bl, g, y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        sharded._unpack(x, bl, g, y)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    ts.sort()
    gbs = 2 * n * 8 / ts[5] / 1e9
    print(json.dumps({"G": G, "per_sm": per_sm, "gbs": round(gbs, 1), "frac": round(gbs / PEAK, 3)}),
          flush=True)
    del x, y
    torch.cuda.empty_cache()
