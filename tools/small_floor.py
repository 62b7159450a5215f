"""Event-timed floor for small launches: torch copy_ vs our out-of-place kernel,
L2 flushed (write + clean read) before each timed launch."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core  # noqa: E402

dev = torch.device("cuda", 0)
w = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
sink = torch.empty((), device=dev)


def timed(fn, reps=30):
    ts = []
    for _ in range(reps):
        w.zero_()
        torch.sum(r, dim=0, out=sink)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for b in (12, 16, 18, 20, 22):
    x = torch.empty(1 << b, dtype=torch.complex128, device=dev).normal_()
    y = torch.empty_like(x)
    t_copy = timed(lambda: y.copy_(x))
    t_ours = timed(lambda: _core.launch_oop(x, y, b))
    t_empty = timed(lambda: None)
    print(f"b={b:2d} bytes={2 * 16 << b:>10d}  empty {t_empty:6.2f} us  copy_ {t_copy:6.2f} us  "
          f"bitrev {t_ours:6.2f} us")
