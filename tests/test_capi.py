"""The C ABI: the library loads, exports every symbol include/bitrev_b200.h
declares, binds them with matching arities, and rejects invalid arguments
before touching CUDA (so these run without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1708_01873_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "bitrev_b200.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    out = {}
    for m in re.finditer(r"^\s*[\w\s\*]+?\b(bitrev_\w+)\s*\(([^)]*)\)\s*;", text, flags=re.M):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else len(args.split(","))
    return out


def test_header_parses():
    names = declared()
    assert "bitrev_oop" in names and "bitrev_inplace" in names
    assert len(names) >= 12


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    for name, arity in declared().items():
        assert hasattr(lib, name), f"{name} declared but not exported"
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
        assert len(_lib.SIGNATURES[name][1]) == arity, name
    assert set(_lib.SIGNATURES) == set(declared())


def test_error_codes_without_gpu():
    lib = _lib.load()
    buf = ctypes.create_string_buffer(1 << 12)
    p = ctypes.addressof(buf)
    assert lib.bitrev_oop(p, p + 2048, 0, 8, 1, 0, 0, None) == -1  # width
    assert lib.bitrev_oop(p, p + 2048, 49, 8, 1, 0, 0, None) == -1
    assert lib.bitrev_oop(p, p + 2048, 4, 3, 1, 0, 0, None) == -2  # element size
    assert lib.bitrev_oop(None, p, 4, 8, 1, 0, 0, None) == -3  # null
    assert lib.bitrev_oop(p, p + 2048, 4, 8, 0, 0, 0, None) == -4  # batch
    assert lib.bitrev_oop(p, p + 2048, 4, 8, 2, 8, 16, None) == -4  # stride < 2^b
    assert lib.bitrev_oop(p, p + 64, 4, 8, 1, 0, 0, None) == -5  # overlap
    assert lib.bitrev_inplace(None, 4, 8, 1, 0, None) == -3
    assert lib.bitrev_inplace(p, 60, 8, 1, 0, None) == -1
    assert lib.bitrev_transpose_square(p, -1, 8, 1, 0, None) == -1
    assert lib.bitrev_sharded_unpack(p, p, 4, 5, 8, None) == -6
    assert lib.bitrev_apply_pairs(p, p, 0, 8, None) == 0  # empty list is a no-op
    assert lib.bitrev_apply_pairs_ordered(p, p, 0, 8, None) == 0
    assert lib.bitrev_apply_pairs_ordered(p, p, -1, 8, None) == -4
    assert lib.bitrev_apply_pairs_ordered(p, None, 3, 8, None) == -3
    assert lib.bitrev_swap_schedule(0, p, None) == -1  # width
    assert lib.bitrev_swap_schedule(49, p, None) == -1
    assert lib.bitrev_swap_schedule(5, None, None) == -3
    assert lib.bitrev_swap_schedule(1, p, None) == 0  # no pairs at width 1
    # sharded pack: width, element size, plan shape (2g + chunk bits <= b_local), overlap
    assert lib.bitrev_sharded_pack(p, p + 2048, 0, 1, 0, 8, None) == -1
    assert lib.bitrev_sharded_pack(p, p + 2048, 10, 1, 0, 2, None) == -2
    assert lib.bitrev_sharded_pack(p, p + 2048, 10, 4, 0, 8, None) == -6  # G = 16 > 8
    assert lib.bitrev_sharded_pack(p, p + 2048, 6, 3, 1, 8, None) == -6
    assert lib.bitrev_sharded_pack(None, p, 10, 1, 0, 8, None) == -3
    assert lib.bitrev_sharded_pack(p, p + 64, 8, 1, 0, 8, None) == -5
    assert lib.bitrev_sharded_scatter(p, None, 10, 1, 0, 8, None) == -3
    assert lib.bitrev_sharded_scatter(p, p, 10, 1, 2, 8, None) == -6  # rank >= G
    for code in (0, -1, -2, -3, -4, -5, -6, -7):
        assert lib.bitrev_strerror(code)
    assert b"overlap" in lib.bitrev_strerror(-5)


def test_tile_bits_registry():
    for E, q_oop, q_ip in ((4, 8, 6), (8, 7, 6), (16, 6, 6)):
        assert _lib.get_tile_bits(E, False) == q_oop
        assert _lib.get_tile_bits(E, True) == q_ip
    _lib.set_tile_bits(8, True, 4)
    assert _lib.get_tile_bits(8, True) == 4
    _lib.set_tile_bits(8, True, 0)
    assert _lib.get_tile_bits(8, True) == 6
    assert _lib.get_tile_order(True) == 2 and _lib.get_tile_order(False) == 0
    for E in (4, 8, 16):
        for ip in (False, True):
            assert _lib.get_tile_path(E, ip) in (0, 1, 2, 3, 4, 5, 6)
    with pytest.raises(_lib.BitrevError):
        _lib.set_tile_bits(8, False, 9)
    with pytest.raises(_lib.BitrevError):
        _lib.set_tile_bits(2, False, 5)


def test_tile_path_registry_and_last_tile():
    """Staging paths: 3 is out-of-place only, 4/5/6 in-place only; defaults
    are the measured ones; bitrev_last_tile rejects NULL outputs."""
    assert [_lib.get_tile_path(E, False) for E in (4, 8, 16)] == [3, 3, 0]
    assert [_lib.get_tile_path(E, True) for E in (4, 8, 16)] == [0, 0, 6]
    for E, ip, path in ((8, True, 3), (8, False, 4), (8, False, 5), (8, False, 6),
                        (8, True, 7), (8, True, -1), (2, True, 0)):
        with pytest.raises(_lib.BitrevError):
            _lib.set_tile_path(E, ip, path)
    for path in (4, 5, 6, 0):
        _lib.set_tile_path(16, True, path)
        assert _lib.get_tile_path(16, True) == path
    _lib.set_tile_path(16, True, 6)
    lib = _lib.load()
    assert lib.bitrev_last_tile(None, None) == -3
    if _lib.launch_count() == 0:  # nothing launched in this process yet: zeros
        assert _lib.last_tile() == (0, 0)


def test_tile_order_registry():
    old = _lib.get_tile_order(True)
    _lib.set_tile_order(True, 1)
    assert _lib.get_tile_order(True) == 1
    _lib.set_tile_order(True, old)
    with pytest.raises(_lib.BitrevError):
        _lib.set_tile_order(False, 7)


def test_version_and_counter():
    assert "sm_100a" in _lib.version()
    assert _lib.launch_count() >= 0


def test_library_targets_sm100a_only():
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out
