"""Batched permutations: many independent rows of length 2^b in one launch.

Extension over the reference (whose functions take one 1-D array,
src/permutations.py:19-24): BASELINE config 4 is the FFT pre-pass over 4096
rows of 2^16 complex64, and one launch over the whole [batch, 2^b] matrix keeps
the grid full where 4096 separate small launches would be launch-bound.
"""

from __future__ import annotations

import torch

from . import _core
from ._core import as_tensor
from .bits import check_width


def _check_rows(t: torch.Tensor, b: int, name: str) -> None:
    check_width(b)
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D [batch, 2**b]")
    if t.shape[1] != (1 << b):
        raise ValueError(f"{name} row length {t.shape[1]} does not match 2**{b}")
    if t.shape[0] < 1:
        raise ValueError(f"{name} needs at least one row")


def bitrev_batched(source, b: int, dest=None) -> torch.Tensor:
    """Out-of-place bit reversal of every row of a [batch, 2^b] tensor.

    Returns dest (allocated like source when not given).
    """
    src = as_tensor(source, "source")
    _check_rows(src, b, "source")
    dst = _core.new_like(src) if dest is None else as_tensor(dest, "dest")
    _check_rows(dst, b, "dest")
    if dst.shape != src.shape or dst.dtype != src.dtype:
        raise ValueError("dest must match source in shape and dtype")
    if _core.shares_memory(src, dst):
        raise ValueError("source and dest must not overlap")
    _core.permute_oop(src, dst, b)
    return dst


def bitrev_batched_inplace(array, b: int) -> None:
    """In-place bit reversal of every row of a [batch, 2^b] tensor."""
    a = as_tensor(array)
    _check_rows(a, b, "array")
    _core.permute_inplace(a, b)
