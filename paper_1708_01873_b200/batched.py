"""Batched permutations: many independent rows of length 2^b in one launch.

Extension over the reference (whose functions take one 1-D array,
src/permutations.py:19-24): BASELINE config 4 is the FFT pre-pass over 4096
rows of 2^16 complex64, and one launch over the whole [batch, 2^b] matrix keeps
the grid full where 4096 separate small launches would be launch-bound.
"""

from __future__ import annotations

import ctypes

import torch

from . import _core, _lib
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


def bitrev_host_pipeline(arrays, b: int, out=None) -> list:
    """Bit-reverse many host arrays through the GPU with overlapped transfers.

    arrays: a sequence of host arrays (torch CPU tensors or numpy arrays), all
    of one shape ([2^b] or [batch, 2^b]) and dtype, contiguous.  out: a
    matching sequence of destination host arrays, or None to permute in place.
    Array k's host->device copy overlaps array k-1's kernel and array k-2's
    device->host copy (bitrev_host_pipeline in the C ABI); pinned host memory
    makes the two copy directions run concurrently.  Synchronous; returns the
    destination list.
    """
    srcs = [as_tensor(a, "arrays[k]") for a in arrays]
    if not srcs:
        return []
    first = srcs[0]
    for t in srcs:
        if t.is_cuda:
            raise ValueError("bitrev_host_pipeline takes host arrays; use the device API for CUDA tensors")
        if t.shape != first.shape or t.dtype != first.dtype:
            raise ValueError("all arrays must share shape and dtype")
        if not t.is_contiguous():
            raise ValueError("arrays must be contiguous")
    if first.dim() == 1:
        from ._core import check_array

        check_array(first, b)
        batch = 1
    else:
        _check_rows(first, b, "arrays[k]")
        batch = first.shape[0]
    dsts = srcs if out is None else [as_tensor(o, "out[k]") for o in out]
    if len(dsts) != len(srcs):
        raise ValueError("out must have one destination per array")
    for d in dsts:
        if d.is_cuda or d.shape != first.shape or d.dtype != first.dtype or not d.is_contiguous():
            raise ValueError("out arrays must be contiguous host arrays shaped like the inputs")
    dev = _core.require_cuda()
    n = len(srcs)
    src_ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in srcs])
    dst_ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in dsts])
    scratch = torch.empty(3 * first.numel() * first.element_size(), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.call("bitrev_host_pipeline", ctypes.cast(src_ptrs, ctypes.c_void_p),
                  ctypes.cast(dst_ptrs, ctypes.c_void_p), n, b, _core.elem_bytes(first), batch,
                  scratch.data_ptr(), _core._stream_ptr(dev))
    return list(out) if out is not None else list(arrays)
