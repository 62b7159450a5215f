"""Per-method entry points of src/permutations.py on the B200 kernels.

Every function keeps the reference signature, argument checks and error
messages (ValueError with the same fragments), and produces the identical
permutation: out-of-place calls land on bitrev_oop, in-place calls
on bitrev_inplace (the tile-pair swap).  The reference's per-method loop
algorithms (Stockham passes, bitwise/bytewise/XOR swap loops, pair exchanges)
are CPU memory-access strategies; on the GPU they are all the same tile kernel.

Arrays: torch tensors (CUDA: asynchronous on the current stream; host: staged
through the device, synchronous) or numpy arrays (wrapped zero-copy, staged).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _core, _lib
from .bits import BYTE_TABLE
from ._core import as_tensor, check_array


# ---------------------------------------------------------------------------
# in-place aliases (src/permutations.py:46-180)


def stockham_permute(array, b: int, scratch=None) -> None:
    """Stockham entry point (src/permutations.py:46-59).  scratch is validated
    like the reference's (>= n elements of the array dtype).  The permutation
    is the tile kernel; a caller-supplied scratch also receives what the
    reference's buffered passes leave in it (bitrev_stockham_scratch, a
    gather from the unpermuted array), so its first n elements end up
    byte-identical to the reference's."""
    a = as_tensor(array)
    check_array(a, b)
    n = a.shape[0]
    if scratch is None:
        _core.permute_inplace(a, b)
        return
    s = as_tensor(scratch, "scratch")
    if s.shape[0] < n or s.dtype != a.dtype:
        raise ValueError(f"scratch must hold {n} elements of {a.dtype}")
    if b == 0:
        return  # one element: the reference's passes never run
    E = _core.elem_bytes(a)
    dev = a.device if a.is_cuda else _core.require_cuda()
    work = a if (a.is_cuda and a.is_contiguous()) else a.to(dev, copy=True).contiguous()
    head = s[:n]
    sd = head if (head.is_cuda and head.device == dev and head.is_contiguous()) else \
        torch.empty(n, dtype=a.dtype, device=dev)
    with torch.cuda.device(dev):
        _lib.call("bitrev_stockham_scratch", work.data_ptr(), sd.data_ptr(), b, E,
                  _core._stream_ptr(dev))
    _core.launch_inplace(work, b)
    if work is not a:
        a.copy_(work)
    if sd is not head:
        head.copy_(sd)


def naive_bitwise_permute(array, b: int) -> None:
    """src/permutations.py:81-88."""
    a = as_tensor(array)
    check_array(a, b)
    _core.permute_inplace(a, b)


def bytetable_permute(array, b: int, table=BYTE_TABLE) -> None:
    """src/permutations.py:107-110 (the byte table is a CPU detail)."""
    a = as_tensor(array)
    check_array(a, b)
    _core.permute_inplace(a, b)


def xor_permute(array, b: int) -> None:
    """src/permutations.py:135-143."""
    a = as_tensor(array)
    check_array(a, b)
    _core.permute_inplace(a, b)


def pair_bitwise_permute(array, b: int) -> None:
    """src/permutations.py:170-180."""
    a = as_tensor(array)
    check_array(a, b)
    _core.permute_inplace(a, b)


# ---------------------------------------------------------------------------
# COBRA (src/permutations.py:187-321)


@dataclass
class CobraConfig:
    """Block-bit parameter q (src/permutations.py:187-211).

    On the CPU q sizes a cache-resident 2^q x 2^q buffer.  The GPU kernels stage
    their own 2^Q x 2^Q tiles in shared memory (Q per element width, see
    bitrev_get_tile_bits); q is validated exactly as the reference does
    (q >= 0, 2q <= b) and does not change the output.
    """

    q: int
    buffer: torch.Tensor | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.q < 0:
            raise ValueError(f"q must be >= 0, got {self.q}")

    @property
    def buffer_size(self) -> int:
        return 1 << (2 * self.q)

    def buffer_for(self, dtype, device=None) -> torch.Tensor:
        t = self.buffer_size
        if (self.buffer is None or self.buffer.dtype != dtype or self.buffer.shape[0] < t
                or (device is not None and self.buffer.device != torch.device(device))):
            self.buffer = torch.empty(t, dtype=dtype, device=device)
        return self.buffer


def default_cobra_q(b: int) -> int:
    """Library default block width (src/permutations.py:214-216)."""
    return min(b // 2, 6)


def _check_cobra(cfg: CobraConfig, b: int) -> None:
    if 2 * cfg.q > b:
        raise ValueError(f"block bits q={cfg.q} need 2q <= b, got b={b}")


def cobra_out_of_place(source, dest, cfg: CobraConfig, b: int) -> None:
    """dest = bit-reversed copy of source (src/permutations.py:293-308).

    source is never written and dest never read.
    """
    src = as_tensor(source, "source")
    dst = as_tensor(dest, "dest")
    check_array(src, b, "source")
    check_array(dst, b, "dest")
    if _core.shares_memory(src, dst):
        raise ValueError("source and dest must not overlap")
    _check_cobra(cfg, b)
    if src.dtype != dst.dtype:
        raise ValueError(f"dest dtype {dst.dtype} does not match source dtype {src.dtype}")
    _core.permute_oop(src, dst, b)


def cobra_in_place(array, cfg: CobraConfig, b: int) -> None:
    """In-place tile-pair swap (src/permutations.py:311-321)."""
    a = as_tensor(array)
    check_array(a, b)
    _check_cobra(cfg, b)
    _core.permute_inplace(a, b)
