"""Run the tile autotuner over every (family, element width) at the BASELINE
sizes on one box; one JSON line per (family, E, b)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200.tune import tune_tiles  # noqa: E402

bits = [int(v) for v in sys.argv[1:]] or [26, 30]
for b in bits:
    for E in (8, 16, 4):
        for ip in (True, False):
            r = tune_tiles(E, ip, b, rounds=5, apply=False)
            print(json.dumps({"b": b, "E": E, "inplace": ip, "best": r.best,
                              "gbs": {f"q{q}p{p}": round(v) for (q, p), v in r.gbs.items()}}),
                  flush=True)
