"""Swap schedules (src/schedule.py): the explicit pair lists that realize the
permutation, and their replay.

A schedule of width b lists every (i, rev i) with i < rev i; swapping the
pairs in any order IS the permutation.  generate_swap_schedule /
cached_schedule return the reference's pair array in its emission order
(_fill_pairs, src/schedule.py:53-91), generated on the device by
bitrev_swap_schedule (one thread per pair, no host loop), as a (count, 2)
int64 CUDA tensor.  save_schedule / load_schedule keep the reference's file
format (src/schedule.py:133-158): the 8-byte magic, one width byte, then the
pairs as little-endian u64.  apply_schedule replays a complete schedule
with the tile kernels (its pairs need not even be materialised), an explicit
disjoint list with the pair kernel, and a list whose pairs share indices in
list order, exactly like _apply_pairs (src/schedule.py:100-107).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np
import torch

from . import _core, _lib
from ._core import as_tensor

SCHEDULE_MAX_BITS = 26
SCHEDULE_MAGIC = b"BRSCHD01"  # schedule file header (src/schedule.py:20)


def swap_count(b: int) -> int:
    """Pairs with i < rev(i): (2^b - 2^ceil(b/2)) / 2 (src/schedule.py:23-37)."""
    if b < 1:
        raise ValueError(f"width must be >= 1, got {b}")
    if b <= 2:
        return b - 1
    return (1 << (b - 2)) + 2 * swap_count(b - 2)


def _device_pairs(b: int, device=None) -> torch.Tensor:
    dev = torch.device(device) if device is not None else _core.require_cuda()
    out = torch.empty((swap_count(b), 2), dtype=torch.int64, device=dev)
    if out.numel():
        with torch.cuda.device(dev):
            _lib.call("bitrev_swap_schedule", b, out.data_ptr(), _core._stream_ptr(dev))
    return out


class SwapSchedule:
    """Width plus the (count, 2) int64 array of (lo, hi) index pairs
    (src/schedule.py:40-51).

    `complete=True` marks the full schedule of width b (what
    generate_swap_schedule / cached_schedule return): its pairs are built on
    the device the first time `.pairs` is read, and apply_schedule runs it as
    the tile-kernel permutation.  A caller-supplied array (numpy or torch) is
    kept as given and replayed pair by pair.
    """

    __slots__ = ("b", "_pairs", "complete")

    def __init__(self, b: int, pairs=None, complete: bool | None = None):
        if pairs is None and complete is False:
            raise ValueError("an incomplete schedule needs its pairs")
        if pairs is not None and (pairs.ndim != 2 or pairs.shape[1] != 2):
            raise ValueError("pairs must have shape (count, 2)")
        self.b = b
        self._pairs = pairs
        self.complete = pairs is None if complete is None else complete

    @property
    def pairs(self):
        if self._pairs is None:
            self._pairs = _device_pairs(self.b)
        return self._pairs

    def __len__(self) -> int:
        return swap_count(self.b) if self._pairs is None else len(self._pairs)

    def __repr__(self) -> str:
        return f"SwapSchedule(b={self.b}, pairs={len(self)}, complete={self.complete})"


def generate_swap_schedule(b: int, max_bits: int = SCHEDULE_MAX_BITS) -> SwapSchedule:
    """All (i, rev i) pairs with i < rev i for width b, in the reference's
    emission order: depth first, the 0-prefix branch before the 1-prefix
    branch, middle values ascending (src/schedule.py:77-91)."""
    if not 1 <= b <= max_bits:
        raise ValueError(f"schedule width must be in 1..{max_bits}, got {b}")
    return SwapSchedule(b, _device_pairs(b), complete=True)


@lru_cache(maxsize=None)
def cached_schedule(b: int) -> SwapSchedule:
    """Shared schedule per width (src/schedule.py:94-97); pairs on first use."""
    if not 1 <= b <= SCHEDULE_MAX_BITS:
        raise ValueError(f"schedule width must be in 1..{SCHEDULE_MAX_BITS}, got {b}")
    return SwapSchedule(b, None, complete=True)


def apply_schedule(array, schedule: SwapSchedule) -> None:
    """Swap every scheduled pair in place (src/schedule.py:124-130)."""
    a = as_tensor(array)
    n = 1 << schedule.b
    if a.shape[0] != n:
        raise ValueError(f"array length {a.shape[0]} does not match 2**{schedule.b}")
    if schedule.complete:
        _core.permute_inplace(a, schedule.b)
        return
    if not a.is_cuda:
        work = a.to(_core.require_cuda())
        apply_schedule(work, schedule)
        a.copy_(work)
        return
    if not a.is_contiguous():
        raise ValueError("apply_schedule with explicit pairs needs a contiguous array")
    p = schedule.pairs
    pairs = (torch.from_numpy(np.array(p, dtype=np.int64)) if isinstance(p, np.ndarray)
             else p.to(torch.int64)).to(a.device).contiguous()
    if pairs.numel() == 0:
        return
    lo, hi = torch.aminmax(pairs)
    if int(lo) < 0 or int(hi) >= n:
        raise ValueError(f"schedule pairs must index [0, 2**{schedule.b})")
    flat = pairs.reshape(-1)
    disjoint = torch.unique(flat).numel() == flat.numel()
    name = "bitrev_apply_pairs" if disjoint else "bitrev_apply_pairs_ordered"
    with torch.cuda.device(a.device):
        _lib.call(name, a.data_ptr(), pairs.data_ptr(), pairs.shape[0], _core.elem_bytes(a),
                  _core._stream_ptr(a.device))


def save_schedule(schedule: SwapSchedule, path) -> None:
    """Write the schedule in the reference's format: magic, width byte, pairs
    as little-endian u64 (src/schedule.py:133-138)."""
    p = schedule.pairs
    arr = p.detach().cpu().numpy() if isinstance(p, torch.Tensor) else np.asarray(p)
    with open(path, "wb") as fh:
        fh.write(SCHEDULE_MAGIC)
        fh.write(bytes([schedule.b]))
        fh.write(np.ascontiguousarray(arr, dtype="<u8").tobytes())


def load_schedule(path) -> SwapSchedule:
    """Read a schedule file (src/schedule.py:141-158): the magic and the pair
    count (swap_count of the stored width) are checked; the pairs come back as
    a read-only host int64 array, replayed as an explicit list."""
    with open(path, "rb") as fh:
        head = fh.read(len(SCHEDULE_MAGIC))
        if head != SCHEDULE_MAGIC:
            raise ValueError(f"{path}: bad magic {head!r}")
        wb = fh.read(1)
        if len(wb) != 1:
            raise ValueError(f"{path}: truncated header")
        body = fh.read()
    b = wb[0]
    words = np.frombuffer(body, dtype="<u8").astype(np.int64)
    want = swap_count(b) if b >= 1 else 0
    if words.size != 2 * want:
        raise ValueError(f"{path}: expected {want} pairs for width {b}, found {words.size // 2}")
    pairs = words.reshape(-1, 2)
    pairs.setflags(write=False)
    return SwapSchedule(b, pairs)
