"""FFT pre-pass on batches of short rows (n*E <= 32 KB: the whole-row FFT
kernel): 2^26 complex64 elements as 2^(26-b) rows of 2^b, GB/s (2*n*E/time)
for 0 stages (plain permutation), a few stages and a complete FFT (b stages)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402

dev = torch.device("cuda", 0)
for dt, E in ((torch.complex64, 8), (torch.complex128, 16)):
    for b in range(4, 13 if E == 8 else 12):
        rows = 1 << (26 - b)
        x = torch.empty(rows, 1 << b, dtype=dt, device=dev)
        x.view(torch.uint8).random_()
        y = torch.empty_like(x)
        res = {"E": E, "b": b}
        for st in sorted({0, 1, 2, min(4, b), b}):
            fn = lambda: br.bitrev_dit_prepass(x, b, st, out=y)  # noqa: E731
            for _ in range(3):
                fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                fn()
            e.record()
            e.synchronize()
            res[f"s{st}"] = round(2 * x.numel() * E / (s.elapsed_time(e) / 1e3 / 10) / 1e9)
        print(json.dumps(res), flush=True)
        del x, y
