"""Size curve: effective GB/s and Gelem/s vs log2 n (BASELINE.json metric), per
element width, in and out of place, beside a streaming comparator of the same
bytes timed in the same harness.

  python tools/size_curve.py [--bits 16 ... 30] [--reps 20] > curve.jsonl

Per cell, one JSON line:
  ours      bitrev (default tile choice) on one array of 2^b elements
  stream    torch copy_ (out of place) / neg_ (in place) of the same bytes
  floor     the event pair around an empty region after the same flush
  batched   for b < 26: rows of 2^b stacked to 2^26 elements, one batched
            launch (the throughput form of small transforms, cfg4-style)

Timing: CUDA events on the current stream, median of `reps`; an L2 flush
(512 MiB write + 256 MiB clean read) precedes every timed launch whose working
set is below 1 GiB, outside the events.
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core  # noqa: E402

DT = {4: torch.float32, 8: torch.float64, 16: torch.complex128}
PEAK = 6551.7  # MEASURED_PEAKS.json hbm_gbs (round 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, nargs="+", default=list(range(16, 31)))
    ap.add_argument("--widths", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
    sink = torch.empty((), device=dev)

    def timed(fn, bytes_moved):
        flush = bytes_moved < (1 << 30)
        fn()
        ts = []
        for _ in range(args.reps):
            if flush:
                w.zero_()
                torch.sum(r, dim=0, out=sink)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e) / 1e3)
        ts.sort()
        return ts[len(ts) // 2]

    t_floor = timed(lambda: None, 0)
    print(json.dumps({"kind": "floor", "us": t_floor * 1e6}), flush=True)
    for E in args.widths:
        for b in args.bits:
            n = 1 << b
            for inplace in (False, True):
                x = torch.empty(n, dtype=DT[E], device=dev)
                x.view(torch.uint8).random_()
                y = None if inplace else torch.empty_like(x)
                moved = 2 * n * E
                if inplace:
                    t = timed(lambda: _core.launch_inplace(x, b), moved)
                    ts = timed(lambda: x.neg_(), moved)
                else:
                    t = timed(lambda: _core.launch_oop(x, y, b), moved)
                    ts = timed(lambda: y.copy_(x), moved)
                rec = {"kind": "cell", "E": E, "b": b, "inplace": inplace, "bytes": moved,
                       "us": t * 1e6, "gbs": moved / t / 1e9, "gelem_s": n / t / 1e9,
                       "frac": moved / t / 1e9 / PEAK, "stream_us": ts * 1e6,
                       "stream_gbs": moved / ts / 1e9, "vs_stream": ts / t}
                del x, y
                if b < 26:
                    rows = 1 << (26 - b)
                    xb = torch.empty(rows, n, dtype=DT[E], device=dev)
                    xb.view(torch.uint8).random_()
                    yb = None if inplace else torch.empty_like(xb)
                    mb = 2 * rows * n * E
                    if inplace:
                        tb = timed(lambda: _core.launch_inplace(xb, b), mb)
                    else:
                        tb = timed(lambda: _core.launch_oop(xb, yb, b), mb)
                    rec.update(batched_rows=rows, batched_gbs=mb / tb / 1e9,
                               batched_frac=mb / tb / 1e9 / PEAK)
                    del xb, yb
                print(json.dumps(rec), flush=True)
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
