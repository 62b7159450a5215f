"""Visit-order sweep for one (kind, b, E, q, path): GB/s per order code,
measured in interleaved rounds so box-to-box drift cancels.

    python tools/order_sweep.py KIND B E Q PATH ORDER [ORDER ...]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402
from paper_1708_01873_b200 import _core  # noqa: E402

kind, b, E, q, path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
orders = [int(o, 0) for o in sys.argv[6:]]
ip = kind == "inplace"
dt = {4: torch.float32, 8: torch.float64, 16: torch.complex128}[E]
dev = torch.device("cuda", 0)
x = torch.empty((1 << b) * E, dtype=torch.uint8, device=dev).random_(0, 256).view(dt)
y = torch.empty_like(x)
br.set_tile_bits(E, ip, q)
br.set_tile_path(E, ip, path)
res = {o: [] for o in orders}
for rnd in range(5):
    for o in orders:
        br.set_tile_order(ip, o)
        fn = (lambda: _core.launch_inplace(x, b)) if ip else (lambda: _core.launch_oop(x, y, b))
        for _ in range(2):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            fn()
        e.record()
        e.synchronize()
        res[o].append(2 * (1 << b) * E * 5 / (s.elapsed_time(e) / 1e3) / 1e9)
for o in orders:
    v = sorted(res[o])
    print(json.dumps({"kind": kind, "b": b, "E": E, "q": q, "path": path, "order": hex(o),
                      "gbs_med": v[len(v) // 2], "gbs_max": v[-1]}), flush=True)
