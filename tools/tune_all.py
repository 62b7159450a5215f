"""Run the tile autotuner over every (family, element width) at the BASELINE
sizes on one box; one JSON line per (family, E, b)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200.tune import tune_tiles  # noqa: E402

import paper_1708_01873_b200 as br  # noqa: E402

args = sys.argv[1:]
families = (True, False)
if "--inplace-only" in args:
    families = (True,)
    args.remove("--inplace-only")
order = None
if "--order" in args:
    i = args.index("--order")
    order = int(args[i + 1], 0)
    del args[i:i + 2]
bits = [int(v) for v in args] or [26, 30]
for b in bits:
    for E in (8, 16, 4):
        for ip in families:
            if order is not None:
                br.set_tile_order(ip, order)
            r = tune_tiles(E, ip, b, rounds=5, apply=False)
            print(json.dumps({"b": b, "E": E, "inplace": ip, "order": br.get_tile_order(ip),
                              "best": r.best,
                              "gbs": {f"q{q}p{p}": round(v) for (q, p), v in r.gbs.items()}}),
                  flush=True)
