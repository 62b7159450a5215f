"""Calibration: HBM GB/s of out-of-place vs in-place streaming ops (torch),
counting 2 bytes moved per byte of array (read + write)."""
import json

import torch

dev = torch.device("cuda", 0)
n = 1 << 28  # 2^28 float32 = 1 GiB
a = torch.empty(n, dtype=torch.float32, device=dev).uniform_()
b = torch.empty_like(a)


def bw(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return 2 * n * 4 * reps / (s.elapsed_time(e) / 1e3) / 1e9


out = {
    "copy_ (oop)": bw(lambda: b.copy_(a)),
    "neg out= (oop)": bw(lambda: torch.neg(a, out=b)),
    "neg_ (in place)": bw(lambda: a.neg_()),
    "mul_ (in place)": bw(lambda: a.mul_(1.0)),
    "copy_ half->half swap view (in place pairs)": None,
}
h = n // 2
t = torch.empty(h, dtype=torch.float32, device=dev)
out["copy_ (oop) again"] = bw(lambda: b.copy_(a))
print(json.dumps(out, indent=1))
