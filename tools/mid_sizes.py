"""Mid-size tile choice: at b = 19..25 a single array has only a few hundred
tiles for 148 SMs, so wave quantisation of the persistent grid matters.  For
every (E, in/out of place, b) this times each instantiated tile width Q (and,
for E=8 out of place, the rectangular path 3) with an L2 flush before every
launch, using the MEAN over many reps: the event timer ticks in ~1.02 us steps
on this pool, and a mean over reps with random phase resolves sub-tick
differences that a median hides.

  python tools/mid_sizes.py [--bits 19 ... 25] [--reps 80] > mid.jsonl
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402

DT = {4: torch.float32, 8: torch.float64, 16: torch.complex128}
QS_OOP = {4: [5, 6, 7], 8: [4, 5, 6, 7], 16: [3, 4, 5, 6]}
QS_IP = {4: [5, 6], 8: [4, 5, 6], 16: [3, 4, 5]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, nargs="+", default=list(range(19, 26)))
    ap.add_argument("--widths", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--reps", type=int, default=80)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
    sink = torch.empty((), device=dev)

    def timed(fn):
        fn()
        tot = 0.0
        for _ in range(args.reps):
            w.zero_()
            torch.sum(r, dim=0, out=sink)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            tot += s.elapsed_time(e) * 1e3
        return tot / args.reps

    print(json.dumps({"kind": "floor_us", "us": timed(lambda: None)}), flush=True)
    for E in args.widths:
        for inplace in (False, True):
            q0 = _lib.get_tile_bits(E, inplace)
            p0 = _lib.get_tile_path(E, inplace)
            for b in args.bits:
                n = 1 << b
                x = torch.empty(n, dtype=DT[E], device=dev)
                x.view(torch.uint8).random_()
                y = None if inplace else torch.empty_like(x)
                run = (lambda: _core.launch_inplace(x, b)) if inplace else \
                      (lambda: _core.launch_oop(x, y, b))
                stream = timed((lambda: x.neg_()) if inplace else (lambda: y.copy_(x)))
                cells = {"default": timed(run)}
                cands = [(q, 0) for q in (QS_IP if inplace else QS_OOP)[E]]
                if E == 8 and not inplace:
                    cands += [(7, 3), (6, 3)]
                if E == 4 and not inplace:
                    cands += [(8, 3), (7, 3)]
                if E == 16 and inplace:
                    cands += [(6, 6), (5, 6)]
                for q, p in cands:
                    if 2 * q > b:
                        continue
                    _lib.set_tile_bits(E, inplace, q)
                    _lib.set_tile_path(E, inplace, p)
                    cells[f"q{q}p{p}"] = timed(run)
                _lib.set_tile_bits(E, inplace, q0)
                _lib.set_tile_path(E, inplace, p0)
                best = min(cells, key=cells.get)
                print(json.dumps({"E": E, "b": b, "inplace": inplace, "stream_us": stream,
                                  "us": cells, "best": best,
                                  "gain_vs_default": cells["default"] / cells[best]}), flush=True)
                del x, y


if __name__ == "__main__":
    main()
