"""A/B of register-tile builds (BITREV_B200_LIB) on the register path."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402
from paper_1708_01873_b200.tune import tune_tiles  # noqa: E402

lib = os.environ.get("BITREV_B200_LIB", "default").split("/")[-1]
for b in (26, 30):
    for E, qs in ((8, (5, 6)), (16, (4, 5, 6)), (4, (5, 6, 7))):
        for ip in (True, False):
            br.set_tile_order(ip, 2 if ip else 0)
            r = tune_tiles(E, ip, b, candidates=[(q, 0) for q in qs], apply=False)
            print(json.dumps({"lib": lib, "b": b, "E": E, "inplace": ip,
                              "gbs": {f"q{q}": round(v) for (q, p), v in r.gbs.items()}}), flush=True)
