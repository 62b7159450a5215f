"""Threaded-variant entry point of src/parallel.py on the B200 kernels.

The reference spreads three barrier-separated phases (block schedules,
transpose tiles, block schedules) over a host thread pool
(src/parallel.py:95-156).  On the GPU the grid is the thread pool and the
permutation is one kernel, so parallel_semi_recursive_permute validates like
the reference and lands on bitrev_inplace.  The static work-plan helpers
(resolve_threads, chunk_ranges, transpose_tiles) are host-side arithmetic kept
with the reference semantics: callers use them to partition work, and the
reference's disjointness tests apply to them unchanged.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

from . import _core
from ._core import as_tensor, check_length
from .recursive import RecursionPolicy, _ensure_scratch

THREADS_ENV = "BITREV_THREADS"
TRANSPOSE_LEAF = 8  # src/recursive.py:27


@dataclass
class ParallelConfig:
    """Worker count and base-case policy (src/parallel.py:32-44)."""

    threads: int = 0
    base_bits: int = 9
    depth_limit: int = 1

    def __post_init__(self):
        if self.threads < 0:
            raise ValueError("threads must be >= 0")
        if self.depth_limit != 1:
            raise ValueError("the parallel variant is defined for depth_limit=1")


def resolve_threads(requested: int = 0) -> int:
    """Explicit request, else BITREV_THREADS, else CPU count (src/parallel.py:47-57)."""
    if requested > 0:
        return requested
    env = os.environ.get(THREADS_ENV)
    if env:
        value = int(env)
        if value < 1:
            raise ValueError(f"{THREADS_ENV} must be >= 1, got {env}")
        return value
    return os.cpu_count() or 1


def chunk_ranges(count: int, workers: int) -> list[tuple[int, int]]:
    """Split range(count) into at most `workers` contiguous chunks (src/parallel.py:60-66)."""
    if count <= 0:
        return []
    workers = max(1, min(workers, count))
    step = -(-count // workers)
    return [(lo, min(lo + step, count)) for lo in range(0, count, step)]


def transpose_tiles(h: int, bands: int = 8) -> list[tuple[str, int, int, int]]:
    """Disjoint tile items covering the 2^h square transposition (src/parallel.py:69-84)."""
    side = 1 << h
    if side <= TRANSPOSE_LEAF or side < bands:
        return [("diag", 0, 0, side)]
    tile = side // bands
    items = []
    for i in range(bands):
        items.append(("diag", i * tile, i * tile, tile))
        for j in range(i + 1, bands):
            items.append(("offdiag", i * tile, j * tile, tile))
    return items


def parallel_semi_recursive_permute(array, b: int, cfg: ParallelConfig | None = None,
                                    scratch=None) -> None:
    """In-place permutation (src/parallel.py:95-156): identical output for any
    thread count; the GPU grid replaces the host pool."""
    a = as_tensor(array)
    check_length(a, b)
    cfg = cfg or ParallelConfig()
    resolve_threads(cfg.threads)  # validates BITREV_THREADS like the reference
    RecursionPolicy(cfg.base_bits, cfg.depth_limit)
    if b > cfg.base_bits and b & 1:
        _ensure_scratch(scratch, a.shape[0] >> 1, a.dtype)
    _core.permute_inplace(a, b)
