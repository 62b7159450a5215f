"""Swap-schedule entry points of src/schedule.py that sit on the hot path.

A complete schedule for width b ({(i, rev i): i < rev i}) applied in any order
IS the permutation, so apply_schedule with a complete schedule takes the tile
kernel; an explicit caller-supplied pair list is replayed by the pair kernel
(bitrev_apply_pairs).  Schedule *generation* (the branch-and-bound _fill_pairs,
the BRSCHD01 file format) is a CPU base-case device of the reference and is out
of scope; swap_count is kept because it is the counting law the
tests pin.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _core, _lib
from ._core import as_tensor

SCHEDULE_MAX_BITS = 26


def swap_count(b: int) -> int:
    """Pairs with i < rev(i): (2^b - 2^ceil(b/2)) / 2 (src/schedule.py:23-37)."""
    if b < 1:
        raise ValueError(f"width must be >= 1, got {b}")
    if b <= 2:
        return b - 1
    return (1 << (b - 2)) + 2 * swap_count(b - 2)


@dataclass(frozen=True)
class SwapSchedule:
    """Width plus an optional (count, 2) int64 pair array.

    pairs=None denotes the complete schedule for width b (what cached_schedule
    returns); an explicit array is replayed pair by pair.
    """

    b: int
    pairs: np.ndarray | torch.Tensor | None = None

    def __post_init__(self):
        if self.pairs is not None and (self.pairs.ndim != 2 or self.pairs.shape[1] != 2):
            raise ValueError("pairs must have shape (count, 2)")

    def __len__(self) -> int:
        return swap_count(self.b) if self.pairs is None else len(self.pairs)


@lru_cache(maxsize=None)
def cached_schedule(b: int) -> SwapSchedule:
    """The complete schedule for width b (src/schedule.py:94-97)."""
    if not 1 <= b <= SCHEDULE_MAX_BITS:
        raise ValueError(f"schedule width must be in 1..{SCHEDULE_MAX_BITS}, got {b}")
    return SwapSchedule(b)


def apply_schedule(array, schedule: SwapSchedule) -> None:
    """Swap every scheduled pair in place (src/schedule.py:124-130)."""
    a = as_tensor(array)
    if a.shape[0] != (1 << schedule.b):
        raise ValueError(f"array length {a.shape[0]} does not match 2**{schedule.b}")
    if schedule.pairs is None:
        _core.permute_inplace(a, schedule.b)
        return
    if not a.is_cuda:
        work = a.to(_core.require_cuda())
        apply_schedule(work, schedule)
        a.copy_(work)
        return
    pairs = torch.as_tensor(schedule.pairs, dtype=torch.int64).to(a.device).contiguous()
    if not a.is_contiguous():
        raise ValueError("apply_schedule with explicit pairs needs a contiguous array")
    with torch.cuda.device(a.device):
        _lib.call("bitrev_apply_pairs", a.data_ptr(), pairs.data_ptr(), pairs.shape[0],
                  _core.elem_bytes(a), _core._stream_ptr(a.device))
