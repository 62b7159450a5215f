"""In-place register pairs against the element-granular cp.async pairs (path 4) at b = 26 / 30 through tune_tiles. Measurement tool."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402
from paper_1708_01873_b200.tune import tune_tiles  # noqa: E402
lib = os.environ.get("BITREV_B200_LIB", "default").split("/")[-1]
br.set_tile_order(True, 2)
for b in (26, 30):
    for E, cands in ((8, [(5, 0), (6, 0), (5, 4), (6, 4)]), (16, [(5, 0), (5, 4), (6, 4)]),
                     (4, [(6, 0), (6, 4), (7, 4)])):
        r = tune_tiles(E, True, b, candidates=cands, apply=False)
        print(json.dumps({"lib": lib, "b": b, "E": E,
                          "gbs": {f"q{q}p{p}": round(v) for (q, p), v in r.gbs.items()}}), flush=True)
