"""Small single arrays (<= 32 MiB per side, the mid-size tiers): register
tiles (the tier default) against the TMA tensor ring (path 2) at the tier's
tile width, L2-flushed (mean over reps: the event timer ticks in ~1 us steps)
and L2-hot (20 launches in one CUDA graph, replayed).  The ring budget is a
build constant: run once on the default library (96 KB, 2 CTAs/SM) and once
on a -DBITREV_RING_BUDGET_KB=200 build (1 CTA/SM, every tile of the SM in
flight) through BITREV_B200_LIB.  Measurement probe only.

  python tools/small_ring_probe.py --tag 96 > out.jsonl
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200 import _core, _lib  # noqa: E402

DT = {4: torch.float32, 8: torch.float64, 16: torch.complex128}
TIER_Q = {4: 5, 8: 4, 16: 5}
BITS = {4: (18, 20, 22, 23), 8: (18, 20, 21, 22), 16: (17, 19, 20, 21)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="96")
    ap.add_argument("--reps", type=int, default=60)
    ap.add_argument("--E", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--bits", type=int, nargs="+", default=None)
    ap.add_argument("--cands", nargs="+", default=None,
                    help="q:path pairs (default: the tier's q with paths 0 and 2)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
    sink = torch.empty((), device=dev)

    def flushed(fn):
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

    def hot(fn, per=20, replays=10):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(per):
                fn()
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(replays):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1e3 / (per * replays)

    for E in args.E:
        cands = ([tuple(int(v) for v in c.split(":")) for c in args.cands] if args.cands
                 else [(TIER_Q[E], 0), (TIER_Q[E], 2)])
        for b in (args.bits or BITS[E]):
            x = torch.empty((1 << b) * E, dtype=torch.uint8, device=dev).random_(0, 256).view(DT[E])
            y = torch.empty_like(x)
            nbytes = 2 * x.numel() * E
            for q, path in cands:
                _lib.set_tile_bits(E, False, q)
                _lib.set_tile_path(E, False, path)
                fn = lambda: _core.launch_oop(x, y, b)  # noqa: E731
                fn()
                used = _lib.last_tile()
                tf, th = flushed(fn), hot(fn)
                print(json.dumps({"budget": args.tag, "E": E, "b": b, "q": q, "path": path, "used": used,
                                  "flushed_us": round(tf, 3), "flushed_gbs": round(nbytes / tf / 1e3, 1),
                                  "hot_us": round(th, 3), "hot_gbs": round(nbytes / th / 1e3, 1)}),
                      flush=True)
            del x, y


if __name__ == "__main__":
    main()
