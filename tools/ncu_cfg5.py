"""One pack (4 exchange rounds) and one unpack of cfg5's G = 8 shard
(b_local = 29 complex64, 4 GiB) for an ncu capture (measurement tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import sharded  # noqa: E402

dev = torch.device("cuda", 0)
bl, g = 29, 3
x = torch.empty((1 << bl) * 8, dtype=torch.uint8, device=dev).random_(0, 256).view(torch.complex64)
y = torch.empty_like(x)
for _ in range(2):
    send = sharded._pack(x, bl, g, 2)
    sharded._unpack(x, bl, g, y)
torch.cuda.synchronize()
print("ok")
