"""FFT pre-pass on rows of 64 KB (complex64 2^13, complex128 2^12): tiles vs the staged-row kernel by stage count. Measurement tool."""
import json, sys, torch
sys.path.insert(0, '/root/repo')
from paper_1708_01873_b200 import _lib
dev = torch.device('cuda', 0)
for dt, E, b in ((torch.complex64, 8, 13), (torch.complex128, 16, 12)):
    rows = 1 << (26 - b)
    x = torch.empty(rows, 1 << b, dtype=dt, device=dev); x.view(torch.uint8).random_()
    y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    res = {"E": E, "b": b}
    for stages in (1, 2, 4, 6, 7, b):
        if E == 16 and stages == 7: continue
        def fn(): _lib.call("bitrev_dit_prepass", x.data_ptr(), y.data_ptr(), b, E, rows, 1 << b, 1 << b, stages, 0, st)
        try:
            for _ in range(3): fn()
        except Exception as e:
            res[f"s{stages}"] = "n/a"; continue
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): fn()
        e.record(); e.synchronize()
        res[f"s{stages}"] = round(2 * x.numel() * E / (s.elapsed_time(e) / 1e3 / 10) / 1e9)
    print(json.dumps(res))
