"""Batched throughput for short rows (the whole-row kernels, n*E <= 32 KB, and
the first tile sizes above): 2^26 elements total as 2^(26-b) rows of 2^b,
out of place and in place, CUDA-event timed (the working set is > L2)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402

dev = torch.device("cuda", 0)
for dt, E in ((torch.float32, 4), (torch.float64, 8), (torch.complex128, 16)):
    bits = [int(x) for x in sys.argv[1:]] or list(range(4, 15))
    for b in bits:
        rows = 1 << (26 - b)
        x = torch.empty(rows, 1 << b, dtype=dt, device=dev)
        x.view(torch.uint8).random_()
        y = torch.empty_like(x)
        res = {"E": E, "b": b, "rows": rows}
        for name, fn in (("oop", lambda: br.bitrev_batched(x, b, y)),
                         ("ip", lambda: br.bitrev_batched_inplace(x, b))):
            for _ in range(3):
                fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                fn()
            e.record()
            e.synchronize()
            t = s.elapsed_time(e) / 1e3 / 10
            res[name] = round(2 * x.numel() * E / t / 1e9)
        res["path"] = br.last_tile()
        print(json.dumps(res), flush=True)
        del x, y
