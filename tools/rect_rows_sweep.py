"""Rectangular out-of-place tiles across row lengths for one element width:
each requested destination-run width QX (path 3; the source-piece width QZ
comes from the library's table or BITREV_B200_RECT_QZ) at 2 GiB per side as
rows of 2^b (batch 2^(31-b-log2 E)... i.e. 2 GiB / row bytes), plus one single
array of 8 GiB.  Median of 20 back-to-back event-timed launches, interleaved
rounds.  Measurement probe only.

  python tools/rect_rows_sweep.py --E 4 --qx 8 9 > out.jsonl
  python tools/rect_rows_sweep.py --E 16 --qx 0 7 > out.jsonl   (0 = library default)
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402

DT = {4: torch.float32, 8: torch.float64, 16: torch.complex128}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=4)
    ap.add_argument("--qx", type=int, nargs="+", default=[8, 9])
    ap.add_argument("--bits", type=int, nargs="+", default=[14, 16, 18, 20, 22, 24, 26])
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    E = args.E
    dev = torch.device("cuda", 0)
    single_b = {4: 31, 8: 30, 16: 29}[E]
    total_b = single_b - 2  # 2 GiB per side for the batched cases
    buf = torch.empty(2 * (E << single_b), dtype=torch.uint8, device=dev)
    cases = [(b, 1 << (total_b - b)) for b in args.bits if b <= total_b] + [(single_b, 1)]
    tag = os.environ.get("BITREV_B200_RECT_QZ", "table")
    default_path = _lib.get_tile_path(E, False)  # qx 0 = the library's default choice
    for rnd in range(args.rounds):
        for b, rows in cases:
            n = rows << b
            x = buf[:E * n].view(DT[E])
            y = buf[E * n:2 * E * n].view(DT[E])
            if rows > 1:
                x, y = x.view(rows, 1 << b), y.view(rows, 1 << b)
            for q in args.qx:
                _lib.set_tile_bits(E, False, q)
                _lib.set_tile_path(E, False, 3 if q else default_path)
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
                print(json.dumps({"round": rnd, "E": E, "qz": tag, "b": b, "rows": rows, "qx": q,
                                  "used": _lib.last_tile(),
                                  "gbs": round(2 * E * n / statistics.median(ts) / 1e9, 1)}),
                      flush=True)


if __name__ == "__main__":
    main()
