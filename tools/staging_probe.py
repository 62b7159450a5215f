"""One staging path of the tile kernels, for an ncu capture and an event
timing (measurement tool; the row-N1 evidence: TMA / cp.async.bulk staging vs
register staging per element width).

    python tools/staging_probe.py E inplace path q b

Prints one JSON line with the event-timed GB/s (median of 10 launches after 3
warm-ups) and the (tile bits, path) the launches actually used."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402

E, inplace, path, q, b = (int(v) for v in sys.argv[1:6])
dt = {4: torch.float32, 8: torch.float64, 16: torch.complex128}[E]
x = torch.empty((1 << b) * E, dtype=torch.uint8, device="cuda").random_(0, 256).view(dt)
y = None if inplace else torch.empty_like(x)
_lib.set_tile_bits(E, bool(inplace), q)
_lib.set_tile_path(E, bool(inplace), path)


def run():
    if inplace:
        _core.launch_inplace(x, b)
    else:
        _core.launch_oop(x, y, b)


for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run()
    e.record()
    e.synchronize()
    ts.append(s.elapsed_time(e) / 1e3)
ts.sort()
used = _lib.last_tile()
print(json.dumps({"E": E, "inplace": bool(inplace), "path": path, "q": q, "b": b,
                  "used": list(used), "gbs": 2 * (1 << b) * E / ts[len(ts) // 2] / 1e9}))
