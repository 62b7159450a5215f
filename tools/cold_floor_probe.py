"""Why does a 16 MiB-per-side copy take ~10 us after an L2 flush but ~4.5 us
L2-hot?  Times torch copy_ and our cfg1 permutation (2^20 complex128) after
different flush recipes, and after the flush plus a TLB-only touch (one
4-byte read per 2 MiB page of src and dst, 64 bytes of DRAM traffic in all),
to separate DRAM latency/bandwidth from address-translation misses.
Measurement probe only."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core  # noqa: E402

dev = torch.device("cuda", 0)
big = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
sink = torch.empty((), device=dev, dtype=torch.float32)
b = 20
x = torch.empty(1 << b, dtype=torch.complex128, device=dev).normal_()
y = torch.empty_like(x)
PAGE = 2 << 20


def touch(t):
    # one element per 2 MiB page: strided view, tiny reduction
    u = t.view(torch.uint8)
    v = u[::PAGE]
    torch.sum(v.to(torch.float32), dim=0, out=sink)


def flush(kind):
    if kind == "none":
        return
    wbytes, rbytes = {"w512r256": (512 << 20, 256 << 20), "w192r192": (192 << 20, 192 << 20),
                      "w1024r512": (1024 << 20, 512 << 20), "w512": (512 << 20, 0)}[kind]
    big[:wbytes].zero_()
    if rbytes:
        # read a region different from the written one where possible
        off = (1 << 30) - rbytes
        torch.sum(big[off:].view(torch.float32), dim=0, out=sink)


def timed(fn, kind, tlb, reps=40):
    ts = []
    for _ in range(reps):
        flush(kind)
        if tlb:
            touch(x)
            touch(y)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


ops = {"copy_": lambda: y.copy_(x), "bitrev": lambda: _core.launch_oop(x, y, b),
       "empty": lambda: None}
for kind in ("w512r256", "w192r192", "w1024r512", "w512", "none"):
    for tlb in (False, True):
        rec = {"flush": kind, "tlb_touch": tlb}
        for name, fn in ops.items():
            fn()
            rec[name + "_us"] = round(timed(fn, kind, tlb), 3)
        print(json.dumps(rec), flush=True)
