"""Timing-only experiment: register kernels with a padded row stride (build
flag BITREV_EXPERIMENT_ROWPAD); the buffer is over-allocated so the padded
rows stay in bounds.  Output is NOT a bit reversal."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402
from paper_1708_01873_b200 import _lib  # noqa: E402

pad = int(os.environ.get("PAD", "0"))
dev = torch.device("cuda", 0)
lib = _lib.load()
for kind, b, E, q in (("inplace", 26, 8, 5), ("inplace", 26, 16, 5), ("oop", 26, 8, 5), ("oop", 26, 16, 6)):
    ip = kind == "inplace"
    br.set_tile_bits(E, ip, q)
    br.set_tile_path(E, ip, 0)
    n = 1 << b
    extra = (pad * (1 << q)) // E + 1024
    x = torch.empty((n + extra) * E, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    def run():
        if ip:
            lib.bitrev_inplace(x.data_ptr(), b, E, 1, 0, st)
        else:
            lib.bitrev_oop(x.data_ptr(), y.data_ptr(), b, E, 1, 0, 0, st)
    res = []
    for _ in range(5):
        run()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            run()
        e.record(); e.synchronize()
        res.append(2 * n * E * 5 / (s.elapsed_time(e) / 1e3) / 1e9)
    res.sort()
    print(json.dumps({"lib": os.environ.get("BITREV_B200_LIB", ""), "pad": pad, "kind": kind, "E": E,
                      "q": q, "gbs_med": round(res[2])}), flush=True)
