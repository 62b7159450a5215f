"""Generate tests/golden/schedule_golden.json by running the REFERENCE's
swap-schedule generator (generate_swap_schedule / _fill_pairs,
/root/reference/pkg/src/bitrev/schedule.py:53-91) for b = 1..22.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_schedule_golden.py

Records the full pair lists for b <= 6 and, for every b, the pair count and
the SHA-256 of the (count, 2) little-endian int64 pair array in emission
order.  Nothing reads /root/reference at test time.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = "/root/reference/pkg/src"


def main() -> None:
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from bitrev.schedule import generate_swap_schedule

    out = {"meta": {"generated_by": "tests/golden/make_schedule_golden.py",
                    "reference": "bitrev.schedule.generate_swap_schedule"},
           "lists": {}, "sha256": {}, "count": {}}
    for b in range(1, 23):
        p = np.ascontiguousarray(generate_swap_schedule(b).pairs, dtype="<i8")
        out["count"][str(b)] = int(p.shape[0])
        out["sha256"][str(b)] = hashlib.sha256(p.tobytes()).hexdigest()
        if b <= 6:
            out["lists"][str(b)] = p.tolist()
    (HERE / "schedule_golden.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
