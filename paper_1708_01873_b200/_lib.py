"""ctypes binding of libbitrev_sm100a.so (the C ABI in include/bitrev_b200.h).

This is the only place the package touches native code.  There is no CPU
fallback: if the library is missing or no CUDA device is visible, every
permutation entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = _PKG_DIR / "libbitrev_sm100a.so"
HEADER_PATH = _PKG_DIR.parent / "include" / "bitrev_b200.h"

_c_int, _c_i64, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p

# name -> (restype, argtypes); must match include/bitrev_b200.h (a CPU test
# parses the header and checks every declared symbol is exported and bound).
SIGNATURES = {
    "bitrev_version": (ctypes.c_char_p, []),
    "bitrev_strerror": (ctypes.c_char_p, [_c_int]),
    "bitrev_oop": (_c_int, [_vp, _vp, _c_int, _c_int, _c_i64, _c_i64, _c_i64, _vp]),
    "bitrev_inplace": (_c_int, [_vp, _c_int, _c_int, _c_i64, _c_i64, _vp]),
    "bitrev_oop_host": (_c_int, [_vp, _vp, _c_int, _c_int, _c_i64, _vp, _vp, _vp]),
    "bitrev_inplace_host": (_c_int, [_vp, _c_int, _c_int, _c_i64, _vp, _vp]),
    "bitrev_host_pipeline": (_c_int, [_vp, _vp, _c_i64, _c_int, _c_int, _c_i64, _vp, _vp]),
    "bitrev_transpose_square": (_c_int, [_vp, _c_int, _c_int, _c_i64, _c_i64, _vp]),
    "bitrev_even_odd": (_c_int, [_vp, _vp, _c_int, _c_int, _c_i64, _c_i64, _c_i64, _vp]),
    "bitrev_stockham_scratch": (_c_int, [_vp, _vp, _c_int, _c_int, _vp]),
    "bitrev_apply_pairs": (_c_int, [_vp, _vp, _c_i64, _c_int, _vp]),
    "bitrev_apply_pairs_ordered": (_c_int, [_vp, _vp, _c_i64, _c_int, _vp]),
    "bitrev_swap_schedule": (_c_int, [_c_int, _vp, _vp]),
    "bitrev_dit_prepass": (_c_int, [_vp, _vp, _c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_int,
                                    _c_int, _vp]),
    "bitrev_dit_prepass_host_pipeline": (_c_int, [_vp, _vp, _c_i64, _c_int, _c_int, _c_i64,
                                                  _c_int, _c_int, _vp, _vp]),
    "bitrev_sharded_scatter": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "bitrev_sharded_pack": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "bitrev_sharded_unpack": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _vp]),
    "bitrev_get_tile_bits": (_c_int, [_c_int, _c_int]),
    "bitrev_set_tile_bits": (_c_int, [_c_int, _c_int, _c_int]),
    "bitrev_get_tile_path": (_c_int, [_c_int, _c_int]),
    "bitrev_set_tile_path": (_c_int, [_c_int, _c_int, _c_int]),
    "bitrev_get_tile_order": (_c_int, [_c_int]),
    "bitrev_set_tile_order": (_c_int, [_c_int, _c_int]),
    "bitrev_launch_count": (_c_i64, []),
    "bitrev_last_tile": (_c_int, [_vp, _vp]),
}

_lock = threading.Lock()
_lib = None


class BitrevError(RuntimeError):
    """A non-zero return code from the native library."""

    def __init__(self, fn: str, code: int, text: str):
        super().__init__(f"{fn} failed ({code}): {text}")
        self.code = code


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and bind the library; raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # BITREV_B200_LIB: load an alternative build (tuning A/B runs only)
        p = Path(path) if path is not None else Path(os.environ.get("BITREV_B200_LIB", LIB_PATH))
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_1708_01873_b200.build` "
                "(bitrev_b200 has no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def call(name: str, *args) -> None:
    """Call an int-returning entry point and raise BitrevError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise BitrevError(name, rc, lib.bitrev_strerror(rc).decode())


def launch_count() -> int:
    return int(load().bitrev_launch_count())


def version() -> str:
    return load().bitrev_version().decode()


def get_tile_bits(elem_bytes: int, inplace: bool) -> int:
    return int(load().bitrev_get_tile_bits(elem_bytes, int(inplace)))


def get_tile_path(elem_bytes: int, inplace: bool) -> int:
    return int(load().bitrev_get_tile_path(elem_bytes, int(inplace)))


def set_tile_path(elem_bytes: int, inplace: bool, path: int) -> None:
    call("bitrev_set_tile_path", elem_bytes, int(inplace), path)


def last_tile() -> tuple[int, int]:
    """(tile bits, staging path) of this thread's most recent bitrev_oop /
    bitrev_inplace launch; path -3 = short-row kernel, -1 = whole-row kernel,
    -2 = element-wise."""
    q, path = ctypes.c_int(0), ctypes.c_int(0)
    call("bitrev_last_tile", ctypes.addressof(q), ctypes.addressof(path))
    return q.value, path.value


def get_tile_order(inplace: bool) -> int:
    return int(load().bitrev_get_tile_order(int(inplace)))


def set_tile_order(inplace: bool, order: int) -> None:
    call("bitrev_set_tile_order", int(inplace), order)


def set_tile_bits(elem_bytes: int, inplace: bool, q: int) -> None:
    call("bitrev_set_tile_bits", elem_bytes, int(inplace), q)
