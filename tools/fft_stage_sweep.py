"""GB/s of the fused FFT pre-pass vs number of fused stages (cfg4 shape)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402
import paper_1708_01873_b200 as br  # noqa: E402

b, rows = 16, 4096
x = torch.empty((rows, 1 << b), dtype=torch.complex64, device="cuda").normal_()
y = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream


def t(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return 2 * x.numel() * 8 * reps / (s.elapsed_time(e) / 1e3) / 1e9


for stages in (0, 1, 2, 4, 6, 7):
    gbs = t(lambda: _lib.call("bitrev_dit_prepass", x.data_ptr(), y.data_ptr(), b, 8, rows,
                              1 << b, 1 << b, stages, 0, st))
    print(f"fft rect stages={stages}: {gbs:.0f} GB/s")
for path, q in ((0, 6), (1, 6), (3, 7)):
    br.set_tile_bits(8, False, q)
    br.set_tile_path(8, False, path)
    print(f"plain bitrev path={path} q={q}: {t(lambda: _core.launch_oop(x, y, b)):.0f} GB/s")
