"""Out-of-place tile-shape probe: source-piece bits QZ of the rectangular
tiles (BITREV_B200_RECT_QZ, read once per process) against the square tiles.

  BITREV_B200_RECT_QZ=5 python tools/rect_qz.py --tag qz5 >> rect.jsonl

Each case: E, QX (tile bits), path (0 square register, 1 bulk ring, 3 rect).
Timing: mean of `reps` back-to-back launches between CUDA events, after 3
warm-up launches; every working set here is >= 512 MiB, above the L2.
"""

import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402

DT = {4: torch.float32, 8: torch.float64, 16: torch.complex128}
CASES = [(4, 7, 0), (4, 7, 3), (4, 8, 3), (8, 6, 1), (8, 6, 3), (8, 7, 3),
         (16, 6, 0), (16, 6, 3), (16, 7, 3)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default=os.environ.get("BITREV_B200_RECT_QZ", "default"))
    ap.add_argument("--bits", type=int, nargs="+", default=[26, 28, 30])
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for b in args.bits:
        for E in sorted({c[0] for c in CASES}):
            n = 1 << b
            x = torch.empty(n, dtype=DT[E], device=dev)
            x.view(torch.uint8).random_()
            y = torch.empty_like(x)
            for E2, q, path in CASES:
                if E2 != E:
                    continue
                _lib.set_tile_bits(E, False, q)
                _lib.set_tile_path(E, False, path)
                for _ in range(3):
                    _core.launch_oop(x, y, b)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(args.reps):
                    _core.launch_oop(x, y, b)
                e.record()
                e.synchronize()
                t = s.elapsed_time(e) / 1e3 / args.reps
                print(json.dumps({"tag": args.tag, "E": E, "b": b, "q": q, "path": path,
                                  "used": list(_lib.last_tile()),
                                  "gbs": 2 * n * E / t / 1e9}), flush=True)
            _lib.set_tile_bits(E, False, 0)
            del x, y
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
