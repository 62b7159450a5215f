"""complex64 FFT pre-pass, 256- vs 128-element destination rows, across
shapes: the QX width is forced per process with BITREV_B200_FFT_QX, so this
prints one line per (shape, stages) for the current setting.  Median of 15
back-to-back event-timed launches.  Measurement probe only.

  BITREV_B200_FFT_QX=8 python tools/fft_qx8_sizes.py > out.jsonl
"""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _lib  # noqa: E402

SHAPES = [(14, 8192), (16, 512), (18, 1024), (20, 64), (22, 64), (24, 16), (26, 4), (28, 1)]
qx = os.environ.get("BITREV_B200_FFT_QX", "auto")
st = torch.cuda.current_stream().cuda_stream
for b, rows in SHAPES:
    x = torch.empty((rows, 1 << b), dtype=torch.complex64, device="cuda").normal_()
    y = torch.empty_like(x)
    for stages in (1, 3, 5, 6, 7):
        fn = lambda: _lib.call("bitrev_dit_prepass", x.data_ptr(), y.data_ptr(), b, 8, rows,  # noqa: E731
                               1 << b, 1 << b, stages, 0, st)
        for _ in range(3):
            fn()
        ts = []
        for _ in range(15):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e) / 1e3)
        print(json.dumps({"qx": qx, "b": b, "rows": rows, "stages": stages,
                          "gbs": round(16 * x.numel() / statistics.median(ts) / 1e9, 1)}), flush=True)
    del x, y
