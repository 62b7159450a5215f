"""Width domain and scalar index reversal (semantics of src/bits.py).

These are host-side helpers on Python ints: they define what the kernels
compute (rev_naive, src/bits.py:31-47) and the accepted widths (check_width,
MAX_BITS, src/bits.py:15-23).  On the device the reversal is one BREV
instruction (`__brevll(i) >> (64 - w)`, csrc/bitrev_kernels.cuh).  The byte
table is kept as a constant because bytetable_permute's signature defaults to
it (src/permutations.py:107).  The reference's other scalar index tricks
(rev_bytetable, count_leading_zeros, the XOR walk RevPair / xor_next,
src/bits.py:59-113) are kept with the same results and errors so code that
calls them keeps working; they are index arithmetic on Python ints, not a
permutation path.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

WORD_BITS = 64
MAX_BITS = 48


def check_width(b: int) -> None:
    """Raise ValueError unless 1 <= b <= MAX_BITS (src/bits.py:21-23)."""
    if not 1 <= b <= MAX_BITS:
        raise ValueError(f"bit width must be in 1..{MAX_BITS}, got {b}")


def _check_index(i: int, b: int) -> None:
    if not 0 <= i < (1 << b):
        raise ValueError(f"index {i} out of range for width {b}")


def rev_naive(i: int, b: int) -> int:
    """Reverse the low b bits of i (src/bits.py:31-47).

    >>> rev_naive(1, 3)
    4
    >>> rev_naive(0b0110, 4)
    6
    """
    check_width(b)
    _check_index(i, b)
    return int(f"{i:0{b}b}"[::-1], 2)


def build_byte_table() -> np.ndarray:
    """256-entry byte-reversal table (src/bits.py:50-56)."""
    table = np.array([int(f"{v:08b}"[::-1], 2) for v in range(256)], dtype=np.uint8)
    table.setflags(write=False)
    return table


BYTE_TABLE = build_byte_table()


def rev_bytetable(i: int, b: int, table: np.ndarray = BYTE_TABLE) -> int:
    """Reverse the low b bits of i with byte-table lookups (src/bits.py:59-72):
    the 64-bit word's bytes are each reversed through the table and laid out
    in the opposite byte order, then shifted down by 64 - b."""
    check_width(b)
    _check_index(i, b)
    word = int.from_bytes(bytes(int(table[v]) for v in i.to_bytes(8, "little")), "big")
    return word >> (WORD_BITS - b)


def count_leading_zeros(x: int) -> int:
    """Zero bits above the highest set bit of a 64-bit word (src/bits.py:75-86);
    undefined (ValueError) for 0 and for values wider than 64 bits."""
    if x == 0:
        raise ValueError("count_leading_zeros is undefined for 0")
    if x >> WORD_BITS:
        raise ValueError(f"{x:#x} does not fit in a 64-bit word")
    return WORD_BITS - x.bit_length()


class RevPair(NamedTuple):
    """An index together with its bit reversal (src/bits.py:89-93)."""

    index: int
    reversed: int


def xor_next(state: RevPair, b: int) -> RevPair:
    """(i, rev i) -> (i + 1, rev(i + 1)) without reversing i + 1
    (src/bits.py:96-113): i ^ (i + 1) is a run of ones from bit 0, and its
    reversal is the same run at the top of the b-bit frame."""
    check_width(b)
    i, r = state
    if not 0 <= i < (1 << b) - 1:
        raise ValueError(f"index {i} cannot be advanced within width {b}")
    if r != rev_naive(i, b):
        raise AssertionError("RevPair is inconsistent")
    run = i ^ (i + 1)
    return RevPair(i + 1, r ^ (run << (b - run.bit_length())))
