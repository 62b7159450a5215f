"""Tensor plumbing between the reference-shaped Python API and the C ABI.

Arrays are torch tensors (numpy arrays are wrapped zero-copy with
torch.from_numpy, so reference callers keep working).  CUDA tensors are
permuted on their own device, enqueued on torch's current stream; host tensors
go through the synchronous *_host entry points (H2D, kernel, D2H) with device
scratch from torch's caching allocator.  Nothing here computes a permutation on
the CPU.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .bits import check_width

ELEM_SIZES = (1, 2, 4, 8, 16)


def as_tensor(x, name: str = "array") -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x
    if isinstance(x, np.ndarray):
        return torch.from_numpy(x)
    raise TypeError(f"{name} must be a torch.Tensor or numpy.ndarray, got {type(x).__name__}")


def check_array(t: torch.Tensor, b: int, name: str = "array") -> None:
    """Mirror of _check_array (src/permutations.py:19-24)."""
    check_width(b)
    if t.dim() != 1:
        raise ValueError(f"{name} must be 1-D")
    if t.shape[0] != (1 << b):
        raise ValueError(f"{name} length {t.shape[0]} does not match 2**{b}")


def check_length(t: torch.Tensor, b: int, name: str = "array") -> None:
    """Mirror of the recursive-module check (src/recursive.py:210-212)."""
    check_width(b)
    if t.dim() != 1 or t.shape[0] != (1 << b):
        raise ValueError(f"{name} length {t.shape[0]} does not match 2**{b}")


def elem_bytes(t: torch.Tensor) -> int:
    e = t.element_size()
    if e not in ELEM_SIZES:
        raise ValueError(f"dtype {t.dtype} has unsupported element size {e}")
    return e


def byte_range(t: torch.Tensor) -> tuple[int, int]:
    if t.numel() == 0:
        return (t.data_ptr(), t.data_ptr())
    extent = sum((s - 1) * st for s, st in zip(t.shape, t.stride()) if s > 0)
    start = t.data_ptr()
    return (start, start + (extent + 1) * t.element_size())


def shares_memory(a: torch.Tensor, b: torch.Tensor) -> bool:
    if a.device != b.device:
        return False
    a0, a1 = byte_range(a)
    b0, b1 = byte_range(b)
    return a0 < b1 and b0 < a1


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("bitrev_b200 needs a CUDA device (B200, sm_100a); it has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _rows(t: torch.Tensor, b: int) -> tuple[int, int]:
    """(batch, batch stride in elements) of a contiguous 1-D or 2-D tensor."""
    if t.dim() == 1:
        return 1, 1 << b
    return t.shape[0], t.stride(0)


# ---------------------------------------------------------------------------
# device launches on contiguous tensors


def launch_oop(src: torch.Tensor, dst: torch.Tensor, b: int) -> None:
    batch, sbs = _rows(src, b)
    _, dbs = _rows(dst, b)
    with torch.cuda.device(src.device):
        _lib.call("bitrev_oop", src.data_ptr(), dst.data_ptr(), b, elem_bytes(src), batch, sbs,
                  dbs, _stream_ptr(src.device))


def launch_inplace(a: torch.Tensor, b: int) -> None:
    batch, bs = _rows(a, b)
    with torch.cuda.device(a.device):
        _lib.call("bitrev_inplace", a.data_ptr(), b, elem_bytes(a), batch, bs,
                  _stream_ptr(a.device))


def _rowwise_ok(t: torch.Tensor) -> bool:
    return t.is_contiguous() or (t.dim() == 2 and t.stride(1) == 1)


# ---------------------------------------------------------------------------
# entry-point bodies (validation happens in the callers)


def permute_inplace(a: torch.Tensor, b: int) -> None:
    """Bit-reverse every row of `a` in place (a: 1-D of 2^b, or 2-D [batch, 2^b])."""
    elem_bytes(a)
    if a.is_cuda:
        if _rowwise_ok(a):
            launch_inplace(a, b)
        else:  # strided view: permute a packed copy, write it back (device copies)
            work = a.contiguous()
            launch_inplace(work, b)
            a.copy_(work)
        return
    dev = require_cuda()
    batch = 1 if a.dim() == 1 else a.shape[0]
    host = a if a.is_contiguous() else a.contiguous()
    buf = torch.empty(host.shape, dtype=host.dtype, device=dev)
    with torch.cuda.device(dev):
        _lib.call("bitrev_inplace_host", host.data_ptr(), b, elem_bytes(host), batch,
                  buf.data_ptr(), _stream_ptr(dev))
    if host is not a:
        a.copy_(host)


def permute_oop(src: torch.Tensor, dst: torch.Tensor, b: int) -> None:
    """dst = bit-reversal of src, row by row (same shapes, dtypes, devices)."""
    elem_bytes(src)
    if src.is_cuda and dst.is_cuda:
        if src.device != dst.device:
            raise ValueError("source and dest must be on the same device")
        s = src if _rowwise_ok(src) else src.contiguous()
        if _rowwise_ok(dst):
            launch_oop(s, dst, b)
        else:
            out = torch.empty(dst.shape, dtype=dst.dtype, device=dst.device)
            launch_oop(s, out, b)
            dst.copy_(out)
        return
    if src.is_cuda != dst.is_cuda:
        raise ValueError("source and dest must both be CUDA tensors or both host arrays")
    dev = require_cuda()
    batch = 1 if src.dim() == 1 else src.shape[0]
    hs = src if src.is_contiguous() else src.contiguous()
    hd = dst if dst.is_contiguous() else torch.empty(dst.shape, dtype=dst.dtype)
    ds = torch.empty(hs.shape, dtype=hs.dtype, device=dev)
    dd = torch.empty(hs.shape, dtype=hs.dtype, device=dev)
    with torch.cuda.device(dev):
        _lib.call("bitrev_oop_host", hs.data_ptr(), hd.data_ptr(), b, elem_bytes(hs), batch,
                  ds.data_ptr(), dd.data_ptr(), _stream_ptr(dev))
    if hd is not dst:
        dst.copy_(hd)


def new_like(t: torch.Tensor) -> torch.Tensor:
    return torch.empty(t.shape, dtype=t.dtype, device=t.device)
