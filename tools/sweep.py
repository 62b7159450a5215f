"""Tile-width sweep on the GPU: effective GB/s of each kernel family per
(element width, tile bits Q, b).  Output: one JSON line per cell.

  python tools/sweep.py [--bits 20 26 30] [--reps 20]

Timing: CUDA events on the current stream around `reps` back-to-back launches
on inputs larger than L2 (or an L2 flush before each launch when the working
set is smaller), after 3 warm-up launches.
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402
from paper_1708_01873_b200 import _core  # noqa: E402

QS = {4: [5, 6, 7], 8: [4, 5, 6, 7], 16: [3, 4, 5, 6]}
DT = {4: torch.float32, 8: torch.float64, 16: torch.complex128}


def time_it(fn, reps, flush=None):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, nargs="+", default=[20, 26, 28])
    ap.add_argument("--widths", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--inplace", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--orders", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--qs", type=int, nargs="*", default=None)
    ap.add_argument("--paths", type=int, nargs="+", default=[0, 1])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    copy_src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    copy_dst = torch.empty_like(copy_src)
    med, best = time_it(lambda: copy_dst.copy_(copy_src), 10)
    print(json.dumps({"kind": "copy_", "bytes": 2 << 30, "gbs_med": 2 * (1 << 30) / med / 1e9,
                      "gbs_best": 2 * (1 << 30) / best / 1e9}), flush=True)
    del copy_src, copy_dst
    for b in args.bits:
        for E in args.widths:
            n = 1 << b
            if 2 * n * E > 40 << 30:
                continue
            src = torch.empty(n * E, dtype=torch.uint8, device=dev).view(DT[E])
            src.view(torch.uint8).random_()
            dst = torch.empty_like(src)
            fl = flush if 2 * n * E < (256 << 20) else None
            for ip in args.inplace:
                for q in (args.qs or QS[E]):
                    if 2 * q > b or q not in QS[E]:
                        continue
                    for order, path in [(o, p) for o in args.orders for p in args.paths]:
                        br.set_tile_bits(E, bool(ip), q)
                        br.set_tile_order(bool(ip), order)
                        br.set_tile_path(E, bool(ip), path)
                        if ip:
                            fn = lambda: _core.launch_inplace(src, b)  # noqa: E731
                        else:
                            fn = lambda: _core.launch_oop(src, dst, b)  # noqa: E731
                        med, best = time_it(fn, args.reps, fl)
                        gb = 2 * n * E / 1e9
                        print(json.dumps({"kind": "inplace" if ip else "oop", "b": b, "E": E,
                                          "q": q, "order": order, "path": path,
                                          "ms_med": med * 1e3,
                                          "gbs_med": gb / med, "gbs_best": gb / best,
                                          "l2_flushed": fl is not None}), flush=True)
                br.set_tile_bits(E, bool(ip), 0)
                br.set_tile_order(bool(ip), 0)
                br.set_tile_path(E, bool(ip), 0)
            del src, dst


if __name__ == "__main__":
    main()
