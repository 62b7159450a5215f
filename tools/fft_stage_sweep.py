"""GB/s of the fused FFT pre-pass vs number of fused stages (cfg4 shape:
4096 rows of 2^16; --c128 for 2048 complex128 rows).  BITREV_B200_FFT_QZ=5
selects 256-byte source pieces for complex64 (A/B runs; round 1's A/B of the
per-stage tile shapes: profiles/r01_fft_qz_ab.txt)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402

C128 = "--c128" in sys.argv
E = 16 if C128 else 8
b, rows = 16, 4096 if not C128 else 2048
x = torch.empty((rows, 1 << b), dtype=torch.complex128 if C128 else torch.complex64,
                device="cuda").normal_()
import os
tag = f"E={E} qz={os.environ.get('BITREV_B200_FFT_QZ', '4')}"
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
    return 2 * x.numel() * E * reps / (s.elapsed_time(e) / 1e3) / 1e9


for stages in (0, 1, 2, 3, 4, 5, 6, 7) if E == 8 else (0, 1, 2, 3, 4, 5, 6):
    gbs = t(lambda: _lib.call("bitrev_dit_prepass", x.data_ptr(), y.data_ptr(), b, E, rows,
                              1 << b, 1 << b, stages, 0, st))
    print(f"{tag} fft rect stages={stages}: {gbs:.0f} GB/s")
print(f"{tag} plain bitrev (default tiles {_lib.get_tile_bits(E, False)}/"
      f"{_lib.get_tile_path(E, False)}): {t(lambda: _core.launch_oop(x, y, b)):.0f} GB/s")
