"""FFT pre-pass: the bit reversal fused with the first radix-2 DIT stages.

The permutation is the first step of an iterative decimation-in-time FFT
(PAPER.md:60-148).  Stages 1..Q of that FFT act inside aligned blocks of 2^Q
outputs, which are exactly the destination rows of the tile kernels, so
bitrev_dit_prepass runs them in the tile drain at the permutation's HBM
traffic: up to 7 stages for complex64, 6 for complex128.
Rows of at most 64 KB take any number of stages, so stages = b gives a
complete (unnormalised) radix-2 FFT.
"""

from __future__ import annotations

import ctypes

import torch

from . import _core, _lib
from ._core import as_tensor
from .bits import check_width

_COMPLEX = {torch.complex64: 8, torch.complex128: 16}


def bitrev_dit_prepass(x, b: int, stages: int, inverse: bool = False, out=None) -> torch.Tensor:
    """Bit-reverse each row of x (complex64/complex128, [2^b] or [batch, 2^b])
    and apply the first `stages` radix-2 DIT butterfly stages, with twiddles
    exp(-2 pi i k / 2^s) (conjugated when inverse; no 1/n scaling).

    Returns out (allocated like x when not given).  CUDA tensors run
    asynchronously on the current stream; host tensors are staged through the
    device.
    """
    t = as_tensor(x, "x")
    check_width(b)
    if t.dtype not in _COMPLEX:
        raise ValueError(f"dtype {t.dtype} is not complex64/complex128")
    if t.dim() not in (1, 2) or t.shape[-1] != (1 << b):
        raise ValueError(f"x length {t.shape[-1]} does not match 2**{b}")
    if not 0 <= stages <= b:
        raise ValueError(f"stages must be in 0..{b}, got {stages}")
    dst = torch.empty_like(t) if out is None else as_tensor(out, "out")
    if dst.shape != t.shape or dst.dtype != t.dtype:
        raise ValueError("out must match x in shape and dtype")
    if _core.shares_memory(t, dst):
        raise ValueError("x and out must not overlap")
    if t.is_cuda:
        dev = t.device
        src_d = t.contiguous()
        # the kernel writes dst_d on x's device: anything else (a host or numpy
        # out, another GPU, a strided view) gets a device temporary copied back
        same = isinstance(dst, torch.Tensor) and dst.device == dev and dst.is_contiguous()
        dst_d = dst if same else torch.empty_like(src_d)
    else:
        dev = _core.require_cuda()
        src_d = t.contiguous().to(dev)
        dst_d = torch.empty_like(src_d)
    batch = 1 if t.dim() == 1 else t.shape[0]
    n = 1 << b
    with torch.cuda.device(dev):
        _lib.call("bitrev_dit_prepass", src_d.data_ptr(), dst_d.data_ptr(), b, _COMPLEX[t.dtype],
                  batch, n, n, stages, int(bool(inverse)), _core._stream_ptr(dev))
    if dst_d is not dst:
        dst.copy_(dst_d)
    return dst


def dit_prepass_host_pipeline(arrays, b: int, stages: int, out=None,
                              inverse: bool = False) -> list:
    """bitrev_dit_prepass over many host arrays with overlapped transfers.

    arrays: host arrays (torch CPU tensors or numpy arrays) of one shape
    ([2^b] or [batch, 2^b]) and complex dtype, contiguous.  out: matching
    destination host arrays, or None to write each result over its input.
    Array k's host->device copy overlaps array k-1's kernel and array k-2's
    device->host copy (bitrev_dit_prepass_host_pipeline in the C ABI); pinned
    host memory lets both copy directions run at once.  Synchronous; returns
    the destination list.
    """
    srcs = [as_tensor(a, "arrays[k]") for a in arrays]
    if not srcs:
        return []
    first = srcs[0]
    if first.dtype not in _COMPLEX:
        raise ValueError(f"dtype {first.dtype} is not complex64/complex128")
    check_width(b)
    if first.dim() not in (1, 2) or first.shape[-1] != (1 << b):
        raise ValueError(f"arrays[k] length {first.shape[-1]} does not match 2**{b}")
    if not 0 <= stages <= b:
        raise ValueError(f"stages must be in 0..{b}, got {stages}")
    for t in srcs:
        if t.is_cuda:
            raise ValueError("dit_prepass_host_pipeline takes host arrays; use "
                             "bitrev_dit_prepass for CUDA tensors")
        if t.shape != first.shape or t.dtype != first.dtype:
            raise ValueError("all arrays must share shape and dtype")
        if not t.is_contiguous():
            raise ValueError("arrays must be contiguous")
    dsts = srcs if out is None else [as_tensor(o, "out[k]") for o in out]
    if len(dsts) != len(srcs):
        raise ValueError("out must have one destination per array")
    for d in dsts:
        if d.is_cuda or d.shape != first.shape or d.dtype != first.dtype or not d.is_contiguous():
            raise ValueError("out arrays must be contiguous host arrays shaped like the inputs")
    dev = _core.require_cuda()
    n = len(srcs)
    batch = 1 if first.dim() == 1 else first.shape[0]
    src_ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in srcs])
    dst_ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in dsts])
    scratch = torch.empty(6 * first.numel() * first.element_size(), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.call("bitrev_dit_prepass_host_pipeline", ctypes.cast(src_ptrs, ctypes.c_void_p),
                  ctypes.cast(dst_ptrs, ctypes.c_void_p), n, b, _COMPLEX[first.dtype], batch,
                  stages, int(bool(inverse)), scratch.data_ptr(), _core._stream_ptr(dev))
    return list(out) if out is not None else list(arrays)


def max_fused_stages(b: int, elem_bytes: int) -> int:
    """Stages the fused path accepts for a row of 2^b elements: all of them
    (a complete FFT) for rows up to 64 KB, else 7 (complex64) / 6
    (complex128)."""
    if (1 << b) * elem_bytes <= 64 * 1024:
        return b
    return 7 if elem_bytes == 8 else 6
