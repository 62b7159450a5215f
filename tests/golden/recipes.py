"""Deterministic input recipes shared by make_golden.py and the tests.

numpy's PCG64 streams are stable across machines, so the GPU box rebuilds the
exact bytes the reference was run on here.
"""

from __future__ import annotations

import numpy as np

BITS_DTYPES = {1: np.uint8, 2: np.int16, 4: np.float32, 8: np.float64, 16: np.complex128}
FILL_KINDS = {"pair": np.complex128, "f8": np.float64, "f4": np.float32, "i8": np.int64}
# method index of "cobra" in METHOD_IDS (src/bench.py:44-56), used as the
# method component of the reference _fill seed
_COBRA_INDEX = 4


_PERM_CACHE: dict = {}


def _perm2024(b: int, trial: int) -> np.ndarray:
    if (b, trial) not in _PERM_CACHE:
        rng = np.random.default_rng(2024)
        for bb in (20, 22, 24):
            for t in range(5):
                x = rng.permutation(1 << bb).astype(np.int64)
                if bb == b and t == trial:
                    _PERM_CACHE.clear()
                    _PERM_CACHE[(b, trial)] = x
                    return x
        raise ValueError(f"perm2024 has no case b={b} trial={trial}")
    return _PERM_CACHE[(b, trial)]


def make_input(recipe: str, E: int, b: int, trial: int = 0) -> np.ndarray:
    n = 1 << b
    if recipe == "bits":
        # raw random bit patterns (NaN payloads, -0.0, denormals included)
        rng = np.random.default_rng([b, E, 7])
        return rng.integers(0, 256, n * E, dtype=np.uint8).view(BITS_DTYPES[E])
    if recipe.startswith("fill:"):
        # the reference benchmark fill (src/bench.py:299-309), seed 0, rep 0
        dtype = np.dtype(FILL_KINDS[recipe[5:]])
        rng = np.random.default_rng(np.random.SeedSequence([0, _COBRA_INDEX, b, 1]))
        out = np.empty(n, dtype=dtype)
        if dtype.kind == "c":
            out.real = rng.standard_normal(n)
            out.imag = rng.standard_normal(n)
        elif dtype.kind == "f":
            out[:] = rng.standard_normal(n, dtype=dtype)
        else:
            out[:] = rng.integers(0, 1 << 62, n, dtype=dtype)
        return out
    if recipe == "perm2024":
        # acceptance-suite inputs (tests/test_acceptance.py:55-58): one
        # default_rng(2024) stream drawn for b in (20, 22, 24) x 5 trials
        return _perm2024(b, trial).copy()
    raise ValueError(f"unknown recipe {recipe!r}")
