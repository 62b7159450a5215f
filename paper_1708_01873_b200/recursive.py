"""Cache-oblivious entry points of src/recursive.py on the B200 kernels.

The paper's method: an even width b splits the index into
halves (hi, lo); reversing each half locally and transposing the 2^(b/2) square
is the whole reversal; odd widths peel off one even-odd pass.  On the GPU the
recursion is flattened: one tile kernel splits the index into (x, y, z) =
(high Q bits, middle, low Q bits) and performs the square transposition of the
(x, z) bits in shared memory while reversing them and the middle bits with BREV,
so every width (odd ones included) is a single pass with one read and one write
per element.  recursive_permute / semi_recursive_permute therefore keep the
reference's signatures, validation and scratch rules, and land on
bitrev_inplace; transpose_square_inplace and even_odd_permute have their own
kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _core, _lib
from ._core import as_tensor, check_length
from .bits import check_width

SCHEDULE_MAX_BITS = 26  # src/schedule.py:17-19


def _ensure_scratch(scratch, needed: int, dtype):
    """Validation of src/recursive.py:110-117 (no allocation: the GPU path
    needs no scratch)."""
    if scratch is None:
        return None
    s = as_tensor(scratch, "scratch")
    if s.shape[0] < needed:
        raise ValueError(f"scratch holds {s.shape[0]} elements, need {needed}")
    if s.dtype != dtype:
        raise ValueError(f"scratch dtype {s.dtype} does not match {dtype}")
    return s


@dataclass
class RecursionPolicy:
    """When the reference stops subdividing (src/recursive.py:120-136)."""

    base_bits: int = 9
    depth_limit: int | None = None

    def __post_init__(self):
        if not 1 <= self.base_bits <= SCHEDULE_MAX_BITS:
            raise ValueError(f"base_bits must be in 1..{SCHEDULE_MAX_BITS}")
        if self.depth_limit is not None and self.depth_limit < 1:
            raise ValueError("depth_limit must be >= 1 when set")


def _hits_base(bb: int, depth: int, policy: RecursionPolicy) -> bool:
    # src/recursive.py:139-149
    if bb <= policy.base_bits:
        return True
    return policy.depth_limit is not None and depth >= policy.depth_limit and bb <= SCHEDULE_MAX_BITS


def _first_odd_width(b: int, policy: RecursionPolicy) -> int | None:
    """Width of the first odd level on the recursion chain, if any.

    All sub-problems at one level share a width, so the chain is a single
    path (src/recursive.py:152-186); the first odd level is where the reference
    validates or allocates its n/2 scratch.
    """
    bb, depth = b, 0
    while not _hits_base(bb, depth, policy):
        if bb & 1:
            return bb
        bb, depth = bb >> 1, depth + 1
    return None


def _plan(off: int, bb: int, depth: int, policy: RecursionPolicy, trace: list) -> None:
    """Append the reference's execution-order events (src/recursive.py:152-186,
    trace path).  Host bookkeeping only: it records the decomposition that the
    single fused GPU pass implements."""
    n = 1 << bb
    if _hits_base(bb, depth, policy):
        trace.append(("base", off, bb))
        return
    if bb & 1:
        trace.append(("even_odd", off, bb))
        _plan(off, bb - 1, depth + 1, policy, trace)
        _plan(off + (n >> 1), bb - 1, depth + 1, policy, trace)
        return
    h = bb >> 1
    m = 1 << h
    for blk in range(m):
        _plan(off + blk * m, h, depth + 1, policy, trace)
    trace.append(("transpose", off, h))
    for blk in range(m):
        _plan(off + blk * m, h, depth + 1, policy, trace)


def recursive_permute(array, b: int, policy: RecursionPolicy | None = None, scratch=None,
                      trace: list | None = None) -> None:
    """Bit-reverse in place (src/recursive.py:189-213).

    scratch is validated by the reference's rule (n/2 elements of the array
    dtype at the first odd level on the chain) and otherwise unused.  trace,
    when given, receives the reference's ("base" | "even_odd" | "transpose",
    offset, width) events for the same policy.
    """
    a = as_tensor(array)
    check_length(a, b)
    policy = policy or RecursionPolicy()
    odd = _first_odd_width(b, policy)
    if odd is not None:
        _ensure_scratch(scratch, 1 << (odd - 1), a.dtype)
    if trace is not None:
        _plan(0, b, 0, policy, trace)
    _core.permute_inplace(a, b)


def semi_recursive_permute(array, b: int, base_bits: int = 9, depth_limit: int = 1,
                           scratch=None) -> None:
    """Depth-limited recursion (src/recursive.py:216-228)."""
    recursive_permute(array, b, RecursionPolicy(base_bits, depth_limit), scratch)


def transpose_square_inplace(region, h: int) -> None:
    """Transpose the 2^h x 2^h row-major matrix stored flat in region
    (src/recursive.py:67-81), one tile-pair kernel."""
    if h < 0:
        raise ValueError(f"h must be >= 0, got {h}")
    r = as_tensor(region, "region")
    if r.dim() != 1 or r.shape[0] != (1 << (2 * h)):
        raise ValueError(f"region length {r.shape[0]} does not match 4**{h}")
    if h == 0:
        return
    if r.is_cuda and r.is_contiguous():
        with torch.cuda.device(r.device):
            _lib.call("bitrev_transpose_square", r.data_ptr(), h, _core.elem_bytes(r), 1,
                      1 << (2 * h), _core._stream_ptr(r.device))
        return
    dev = r.device if r.is_cuda else _core.require_cuda()
    work = r.to(dev, copy=True).contiguous()
    with torch.cuda.device(dev):
        _lib.call("bitrev_transpose_square", work.data_ptr(), h, _core.elem_bytes(work), 1,
                  1 << (2 * h), _core._stream_ptr(dev))
    r.copy_(work)


def even_odd_permute(array, b: int, scratch=None) -> None:
    """Evens to the bottom half, odds to the top (src/recursive.py:96-107).

    The reference parks the odds in an n/2 scratch.  On the device the split
    is the index rotation i -> (i >> 1) | ((i & 1) << (b - 1)), which factors
    into two bit reversals: the full width, then each half (rev_{b-1} on the
    low b-1 bits after rev_b puts bit 0 on top).  Both run in place on the
    tile kernels with no n-element temporary.  A caller-supplied scratch is
    validated like the reference's and, like the reference's, ends up
    holding the odd elements (the new top half) in its first n/2 slots.
    """
    check_width(b)
    a = as_tensor(array)
    if a.dim() != 1 or a.shape[0] != (1 << b):
        raise ValueError(f"array length {a.shape[0]} does not match 2**{b}")
    s = _ensure_scratch(scratch, a.shape[0] >> 1, a.dtype)
    if b == 1:  # [a0, a1] is already split; the reference parks a1
        if s is not None:
            s[:1].copy_(a[1:])
        return
    _core.elem_bytes(a)
    on_device = a.is_cuda and a.is_contiguous()
    dev = a.device if a.is_cuda else _core.require_cuda()
    work = a if on_device else a.to(dev, copy=True).contiguous()  # host / strided: staged once
    _core.launch_inplace(work, b)
    _core.launch_inplace(work.view(2, -1), b - 1)
    if work is not a:
        a.copy_(work)
    if s is not None:  # the reference's parked odds (src/recursive.py:88-89)
        half = a.shape[0] >> 1
        s[:half].copy_(work[half:])
