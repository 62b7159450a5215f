"""Out-of-place defaults vs size: interleaved candidates at several (b, batch)
shapes of ~1-4 GiB, per element width."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1708_01873_b200.tune import tune_tiles  # noqa: E402

C = {4: [(7, 0), (6, 0), (8, 3), (7, 3), (6, 2)], 8: [(6, 1), (5, 0), (7, 3), (6, 3), (6, 2)],
     16: [(6, 0), (5, 1), (7, 3), (6, 3), (4, 1)]}
for E in (8, 4, 16):
    for b, batch in ((16, 4096 * 8 // E), (20, 256 * 8 // E), (24, 16 * 8 // E), (28, 1), (30, 1)):
        cands = [c for c in C[E] if (c[1] == 3 and c[0] + 5 <= b) or (c[1] != 3 and 2 * c[0] <= b)]
        r = tune_tiles(E, False, b, candidates=cands, apply=False, batch=batch)
        print(json.dumps({"E": E, "b": b, "batch": batch,
                          "gbs": {f"q{q}p{p}": round(v) for (q, p), v in r.gbs.items()}}), flush=True)
