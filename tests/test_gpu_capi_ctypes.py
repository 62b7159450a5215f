"""The C ABI driven exactly as INTEGRATION.md's ctypes stub does it: plain
ctypes on numpy arrays, host entry points, NULL device scratch, no torch."""

import ctypes

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1708_01873_b200._lib import LIB_PATH

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib(cuda):
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.bitrev_oop_host.argtypes = [vp, vp, i, i, i64, vp, vp, vp]
    L.bitrev_inplace_host.argtypes = [vp, i, i, i64, vp, vp]
    L.bitrev_strerror.restype = ctypes.c_char_p
    return L


@pytest.mark.parametrize("E,dt", [(4, np.float32), (8, np.float64), (16, np.complex128),
                                  (2, np.int16), (1, np.uint8)])
@pytest.mark.parametrize("b", [3, 12, 17, 21])
def test_stub_copy_and_swap(lib, E, dt, b):
    x = np.random.default_rng(b * 17 + E).integers(0, 256, (1 << b) * E, dtype=np.uint8).view(dt)
    expected = orc.oracle_permute(x, b).view(np.uint8)
    dst = np.empty_like(x)
    assert lib.bitrev_oop_host(x.ctypes.data, dst.ctypes.data, b, E, 1, None, None, None) == 0
    assert np.array_equal(dst.view(np.uint8), expected)
    a = x.copy()
    assert lib.bitrev_inplace_host(a.ctypes.data, b, E, 1, None, None) == 0
    assert np.array_equal(a.view(np.uint8), expected)


def test_stub_reports_errors(lib):
    x = np.zeros(16, dtype=np.float64)
    rc = lib.bitrev_inplace_host(x.ctypes.data, 60, 8, 1, None, None)
    assert rc < 0 and b"width" in lib.bitrev_strerror(rc)


@pytest.mark.parametrize("E,dt", [(8, np.float64), (16, np.complex128), (4, np.float32)])
@pytest.mark.parametrize("b,batch,count", [(14, 1, 5), (20, 1, 4), (12, 3, 7)])
def test_host_pipeline(cuda, E, dt, b, batch, count):
    import torch

    import paper_1708_01873_b200 as br

    rng = np.random.default_rng(b + 100 * E + count)
    arrays = [rng.integers(0, 256, (1 << b) * E * batch, dtype=np.uint8).view(dt).reshape(
        (batch, 1 << b) if batch > 1 else (1 << b,)) for _ in range(count)]
    expected = [np.ascontiguousarray(orc.oracle_permute(a, b)) for a in arrays]
    # out of place into numpy destinations
    outs = [np.empty_like(a) for a in arrays]
    br.bitrev_host_pipeline(arrays, b, outs)
    for o, e in zip(outs, expected):
        assert np.array_equal(o.view(np.uint8), e.view(np.uint8))
    # in place on pinned torch tensors, with the same host array repeated
    pinned = [torch.from_numpy(a.copy()).pin_memory() for a in arrays[:2]]
    seq = [pinned[k % 2] for k in range(4)]
    br.bitrev_host_pipeline(seq, b)  # each array permuted twice -> identity
    for p, a in zip(pinned, arrays[:2]):
        assert np.array_equal(p.numpy().view(np.uint8), a.view(np.uint8))


def test_host_pipeline_pageable_in_place(cuda):
    """numpy (pageable) arrays through bitrev_host_pipeline in place take the
    staged single-call path; a repeated array is permuted twice (identity)."""
    import paper_1708_01873_b200 as br

    b = 22
    rng = np.random.default_rng(5)
    arrays = [rng.integers(0, 1 << 62, 1 << b, dtype=np.int64) for _ in range(2)]
    keep = [a.copy() for a in arrays]
    br.bitrev_host_pipeline([arrays[0], arrays[1], arrays[0]], b)
    assert np.array_equal(arrays[0], keep[0])
    assert np.array_equal(arrays[1], orc.oracle_permute(keep[1], b))
