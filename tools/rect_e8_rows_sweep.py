"""float64 out of place, rectangular tiles: 1 KB (QX = 7) vs 2 KB (QX = 8)
destination rows across row lengths, at 2 GiB per side (rows of 2^b, batch
2^(28-b)) and the 8 GiB single array of cfg3-8.  Median of 20 back-to-back
event-timed launches, interleaved rounds.  Measurement probe only.

  python tools/rect_e8_rows_sweep.py > out.jsonl
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402

CASES = [(b, 1 << (28 - b)) for b in (13, 14, 15, 16, 17, 18, 20, 22, 24, 26)] + [(28, 1), (30, 1)]


def main():
    dev = torch.device("cuda", 0)
    buf = torch.empty(2 * (8 << 30), dtype=torch.uint8, device=dev)
    for rnd in range(3):
        for b, rows in CASES:
            n = rows << b
            x = buf[:8 * n].view(torch.float64).view(rows, 1 << b) if rows > 1 else buf[:8 * n].view(torch.float64)
            y = buf[8 * n:16 * n].view(torch.float64).view(rows, 1 << b) if rows > 1 else buf[8 * n:16 * n].view(torch.float64)
            for q in (7, 8):
                _lib.set_tile_bits(8, False, q)
                _lib.set_tile_path(8, False, 3)
                for _ in range(3):
                    _core.launch_oop(x, y, b)
                ts = []
                for _ in range(20):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    _core.launch_oop(x, y, b)
                    e.record()
                    e.synchronize()
                    ts.append(s.elapsed_time(e) / 1e3)
                print(json.dumps({"round": rnd, "b": b, "rows": rows, "qx": q, "used": _lib.last_tile(),
                                  "gbs": round(16 * n / statistics.median(ts) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
