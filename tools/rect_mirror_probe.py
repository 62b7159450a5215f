"""float64 out of place, rectangular tiles at QX = 5 / 6 / 7 (b = 26 / 28 / 30), 20 back-to-back launches. Measurement tool."""
import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_1708_01873_b200 import _core, _lib
E, dev = 8, torch.device('cuda', 0)
for b in (26, 28, 30):
    x = torch.empty(1 << b, dtype=torch.float64, device=dev); x.view(torch.uint8).random_()
    y = torch.empty_like(x)
    for q in (5, 6, 7):
        _lib.set_tile_bits(E, False, q); _lib.set_tile_path(E, False, 3)
        for _ in range(3): _core.launch_oop(x, y, b)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20): _core.launch_oop(x, y, b)
        e.record(); e.synchronize()
        print(json.dumps({"b": b, "qx": q, "used": _lib.last_tile(), "gbs": round(2 * (1 << b) * E / (s.elapsed_time(e) / 1e3 / 20) / 1e9)}))
    del x, y
