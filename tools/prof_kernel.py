"""Run one tile-kernel configuration a few times (for ncu -s/-c targeting).

    python tools/prof_kernel.py KIND B E Q [ORDER] [REPS] [PATH]   KIND = oop | inplace
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402
from paper_1708_01873_b200 import _core  # noqa: E402

kind, b, E, q = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
order = int(sys.argv[5]) if len(sys.argv) > 5 else 0
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
path = int(sys.argv[7]) if len(sys.argv) > 7 else 0
dt = {4: torch.float32, 8: torch.float64, 16: torch.complex128}[E]
dev = torch.device("cuda", 0)
x = torch.empty((1 << b) * E, dtype=torch.uint8, device=dev).random_(0, 256).view(dt)
y = torch.empty_like(x)
ip = kind == "inplace"
br.set_tile_bits(E, ip, q)
br.set_tile_order(ip, order)
br.set_tile_path(E, ip, path)
for _ in range(reps):
    if ip:
        _core.launch_inplace(x, b)
    else:
        _core.launch_oop(x, y, b)
torch.cuda.synchronize()
print("ok", kind, b, E, q, order)
