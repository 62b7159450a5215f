"""Generate tests/golden/scratch_golden.json by running the REFERENCE package:
the contents a caller-supplied scratch buffer holds after stockham_permute
(/root/reference/pkg/src/bitrev/permutations.py:30-59) and even_odd_permute
(/root/reference/pkg/src/bitrev/recursive.py:84-107).  Both leave
deterministic data there (the last writes of their buffered passes), so a
drop-in that is handed the same scratch reproduces it.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_scratch_golden.py

Each case: the recipe input (recipes.make_input), a scratch of n (+ 5 spare)
elements pre-filled with a fixed byte pattern, SHA-256 of the array and of
the whole scratch after the call.  Nothing reads /root/reference at test time.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from recipes import make_input  # noqa: E402

REF_SRC = "/root/reference/pkg/src"
SPARE = 5


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def scratch_for(x: np.ndarray, n: int) -> np.ndarray:
    raw = np.full((n + SPARE) * x.itemsize, 0xA5, dtype=np.uint8)
    return raw.view(x.dtype)


def main() -> None:
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import numba
    import bitrev as ref

    t0 = time.time()
    cases = []
    for E in (1, 2, 4, 8, 16):
        for b in (1, 2, 3, 5, 8, 11, 14):
            x = make_input("bits", E, b)
            n = 1 << b
            for method in ("stockham", "even_odd"):
                a = x.copy()
                s = scratch_for(x, n if method == "stockham" else n // 2)
                if method == "stockham":
                    ref.stockham_permute(a, b, s)
                else:
                    ref.even_odd_permute(a, b, s)
                cases.append({"method": method, "recipe": "bits", "E": E, "b": b,
                              "scratch_len": int(s.shape[0]), "array_sha256": sha(a),
                              "scratch_sha256": sha(s)})
                print(f"{method:9s} E={E:2d} b={b:2d}", flush=True)
    doc = {"meta": {"generated_by": "tests/golden/make_scratch_golden.py",
                    "reference": "/root/reference/pkg/src/bitrev (bitrev 0.1.0)",
                    "numpy": np.__version__, "numba": numba.__version__,
                    "scratch_fill": "0xA5 bytes, SPARE = 5 extra elements past the needed length",
                    "seconds": round(time.time() - t0, 1)},
           "cases": cases}
    (HERE / "scratch_golden.json").write_text(json.dumps(doc, indent=1) + "\n")
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    main()
