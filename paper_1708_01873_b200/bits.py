"""Width domain and scalar index reversal (semantics of src/bits.py).

These are host-side helpers on Python ints: they define what the kernels
compute (rev_naive, src/bits.py:31-47) and the accepted widths (check_width,
MAX_BITS, src/bits.py:15-23).  On the device the reversal is one BREV
instruction (`__brevll(i) >> (64 - w)`, csrc/bitrev_kernels.cuh).  The byte
table is kept as a constant because bytetable_permute's signature defaults to
it (src/permutations.py:107); the CPU-only index tricks (rev_bytetable, clz,
the XOR walk) have no GPU role and are out of scope.
"""

from __future__ import annotations

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
