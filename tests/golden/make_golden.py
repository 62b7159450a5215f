"""Generate tests/golden/golden.json by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

For every (input recipe, b) it runs all 11 reference methods through
bitrev.make_method (/root/reference/pkg/src/bitrev/bench.py:135-185) and the
reference oracle (verify.py:34-39), requires all 12 outputs to agree byte for
byte, and records SHA-256 digests of the input and output bytes.  The GPU
tests rebuild the input from the same recipe, run the B200 kernels and compare
digests; the CPU tests check the oracle restatement against the same digests.
Nothing reads /root/reference at test time.
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


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def main() -> None:
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import numba
    import bitrev as ref

    def run(method, x, b):
        a = x.copy()
        out = ref.make_method(method)(a, b)
        return a if out is None else out

    t0 = time.time()
    cases = []
    # recipe grid: random bit patterns for every element width, plus the
    # reference's own _fill distributions and acceptance permutations
    grid = []
    for E in (1, 2, 4, 8, 16):
        for b in range(1, 21):
            grid.append(("bits", E, b, 0))
    for E in (4, 8, 16):
        for b in (22, 24):
            grid.append(("bits", E, b, 0))
    for kind in ("pair", "f8", "f4", "i8"):
        for b in (3, 8, 13, 16, 20):
            grid.append((f"fill:{kind}", 0, b, 0))
    for b in (20, 22, 24):
        for trial in range(5):
            grid.append(("perm2024", 8, b, trial))

    all_methods = list(ref.METHOD_IDS)
    for recipe, E, b, trial in grid:
        x = make_input(recipe, E, b, trial)
        expected = ref.oracle_permute(x, b)
        methods = all_methods if b <= 20 else ["cobra", "cobra_inplace", "semirecursive",
                                               "parallel", "xor"]
        for m in methods:
            got = run(m, x, b)
            if sha(got) != sha(expected):
                raise SystemExit(f"reference method {m} disagrees with its oracle: {recipe} b={b}")
        cases.append({
            "recipe": recipe, "E": int(x.itemsize), "b": b, "trial": trial,
            "dtype": str(x.dtype), "input_sha256": sha(x), "output_sha256": sha(expected),
            "reference_methods_agreeing": ["oracle_permute"] + methods,
        })
        print(f"{recipe:12s} E={x.itemsize:2d} b={b:2d} t={trial} ok", flush=True)

    canonical = {m: run(m, np.arange(8, dtype=np.int64), 3).tolist() for m in all_methods}
    small = {str(b): ref.rev_index_array(b).tolist() for b in range(0, 9)}
    transpose = {}
    for h in range(0, 5):
        side = 1 << h
        a = np.random.default_rng(h).permutation(side * side)
        w = a.copy()
        ref.transpose_square_inplace(w, h)
        transpose[str(h)] = {"input": a.tolist(), "output": w.tolist()}
    eo = np.arange(16, dtype=np.int64)
    ref.even_odd_permute(eo, 4)
    doc = {
        "meta": {
            "generated_by": "tests/golden/make_golden.py",
            "reference": "/root/reference/pkg/src/bitrev (bitrev 0.1.0)",
            "numpy": np.__version__, "numba": numba.__version__,
            "seconds": round(time.time() - t0, 1),
            "note": "digests are SHA-256 of raw element bytes (C order)",
        },
        "canonical": canonical,
        "rev_index_small": small,
        "transpose_square": transpose,
        "even_odd_b4": eo.tolist(),
        "swap_count": {str(b): ref.swap_count(b) for b in range(1, 27)},
        "cases": cases,
    }
    (HERE / "golden.json").write_text(json.dumps(doc, indent=1) + "\n")
    print(f"wrote {len(cases)} cases in {doc['meta']['seconds']} s")


if __name__ == "__main__":
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    main()
