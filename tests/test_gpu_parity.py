"""GPU parity: every kernel path vs the CPU oracle, byte for byte.

Inputs are seeded random BIT PATTERNS (numpy default_rng bytes), so any
misplaced element, torn vector or swapped half shows up; comparison is on the
raw bytes (np.array_equal would hide -0.0/NaN differences).
"""

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

DTYPES = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64, 16: torch.complex128}
NP_DTYPES = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64, 16: np.complex128}


def rand_bits(n, E, seed, batch=None):
    rng = np.random.default_rng(seed)
    shape = (n,) if batch is None else (batch, n)
    raw = rng.integers(0, 256, size=(int(np.prod(shape)) * E,), dtype=np.uint8)
    return raw.view(NP_DTYPES[E]).reshape(shape)


def as_bytes(x):
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().contiguous().numpy()
    return np.ascontiguousarray(x).view(np.uint8)


def assert_same(got, expected):
    g, e = as_bytes(got), as_bytes(expected)
    assert g.shape == e.shape
    if not np.array_equal(g, e):
        bad = np.nonzero(g != e)[0]
        pytest.fail(f"{bad.size} bytes differ, first at byte {bad[:4].tolist()}")


WIDTHS = list(range(1, 23))


@pytest.mark.parametrize("E", [4, 8, 16, 2, 1])
@pytest.mark.parametrize("b", WIDTHS)
def test_oop_matches_oracle(cuda, E, b):
    host = rand_bits(1 << b, E, seed=1000 * E + b)
    src = torch.from_numpy(host).to(cuda)
    dst = torch.empty_like(src)
    br.cobra_out_of_place(src, dst, br.CobraConfig(br.default_cobra_q(b)), b)
    torch.cuda.synchronize()
    assert_same(dst, orc.oracle_permute(host, b))
    assert_same(src, host)  # source never written


@pytest.mark.parametrize("E", [4, 8, 16, 2, 1])
@pytest.mark.parametrize("b", WIDTHS)
def test_inplace_matches_oracle(cuda, E, b):
    host = rand_bits(1 << b, E, seed=2000 * E + b)
    a = torch.from_numpy(host).to(cuda)
    br.cobra_in_place(a, br.CobraConfig(br.default_cobra_q(b)), b)
    torch.cuda.synchronize()
    assert_same(a, orc.oracle_permute(host, b))


@pytest.mark.parametrize("E", [4, 8, 16])
@pytest.mark.parametrize("b", [16, 17, 20, 21])
def test_every_tile_size(cuda, E, b):
    """Every instantiated tile width Q gives the same bytes (output never
    depends on the tile parameter, like CobraConfig.q)."""
    host = rand_bits(1 << b, E, seed=3000 * E + b)
    expected = orc.oracle_permute(host, b)
    qs = {4: [5, 6, 7], 8: [4, 5, 6], 16: [3, 4, 5, 6]}[E]
    orders = [br.get_tile_order(False), br.get_tile_order(True)]
    paths = [br.get_tile_path(E, False), br.get_tile_path(E, True)]
    try:
        for q in qs:
            for order in (0, 1, 2):
                for path in (0, 1, 2, 4, 5, 6):
                    for inplace in (False, True):
                        br.set_tile_bits(E, inplace, q)
                        br.set_tile_order(inplace, order)
                        br.set_tile_path(E, inplace, path if (inplace or path < 4) else 0)
                    src = torch.from_numpy(host).to(cuda)
                    dst = torch.empty_like(src)
                    br.cobra_out_of_place(src, dst, br.CobraConfig(0), b)
                    br.cobra_in_place(src, br.CobraConfig(0), b)
                    torch.cuda.synchronize()
                    assert_same(dst, expected)
                    assert_same(src, expected)
    finally:
        for inplace in (False, True):
            br.set_tile_bits(E, inplace, 0)
            br.set_tile_order(inplace, orders[int(inplace)])
            br.set_tile_path(E, inplace, paths[int(inplace)])


@pytest.mark.parametrize("E,q", [(4, 6), (4, 7), (4, 8), (8, 5), (8, 6), (8, 7),
                                 (16, 4), (16, 5), (16, 6), (16, 7)])
@pytest.mark.parametrize("b,batch", [(12, 3), (13, 2), (17, 1), (21, 2)])
def test_rect_out_of_place_tiles(cuda, E, q, b, batch):
    """Rectangular out-of-place tiles (path 3), including widths below QX+QZ
    (the dispatcher then falls back to square tiles)."""
    host = rand_bits(1 << b, E, seed=7000 * E + 10 * b + q, batch=batch)
    expected = orc.oracle_permute(host, b)
    old = (br.get_tile_bits(E, False), br.get_tile_path(E, False))
    try:
        br.set_tile_bits(E, False, q)
        br.set_tile_path(E, False, 3)
        out = br.bitrev_batched(torch.from_numpy(host).to(cuda), b)
        torch.cuda.synchronize()
        assert_same(out, expected)
    finally:
        br.set_tile_bits(E, False, old[0])
        br.set_tile_path(E, False, old[1])


@pytest.mark.parametrize("E", [4, 8, 16])
@pytest.mark.parametrize("b,batch", [(2, 4097), (3, 1000), (5, 3), (7, 2049), (9, 130),
                                     (11, 17), (12, 5), (13, 3)])
@pytest.mark.parametrize("pad", [0, 16])
def test_short_rows_kernel(cuda, E, b, batch, pad):
    """Short rows (n*E <= 32 KB): many rows per CTA, partial last blocks,
    padded row strides, in and out of place."""
    if (E << b) > 32 * 1024 or (E << b) < 16:
        pytest.skip("not a short-row case")
    n = 1 << b
    host = rand_bits((n + pad) * batch, E, seed=9000 + 100 * E + b).reshape(batch, n + pad)
    expected = orc.oracle_permute(np.ascontiguousarray(host[:, :n]), b)
    buf = torch.from_numpy(host.copy()).to(cuda)
    rows = buf[:, :n]
    out = torch.zeros(batch, n, dtype=buf.dtype, device=cuda)
    br.bitrev_batched(rows, b, out)
    assert br.last_tile() == (0, -3)
    br.bitrev_batched_inplace(rows, b)
    assert br.last_tile() == (0, -3)
    torch.cuda.synchronize()
    assert_same(out, expected)
    assert_same(rows.contiguous(), expected)
    if pad:  # padding between rows untouched
        assert_same(buf[:, n:].contiguous(), np.ascontiguousarray(host[:, n:]))


@pytest.mark.parametrize("E,b,batch", [(4, 14, 1024), (8, 13, 1024), (8, 14, 513),
                                       (16, 12, 1025), (16, 13, 512)])
def test_inplace_mid_rows_in_large_batches(cuda, E, b, batch):
    """In place, rows of 64-128 KB in batches of >= 64 MiB take the short-row
    kernel with one row per block (a whole row staged in one CTA)."""
    n = 1 << b
    pad = 16
    host = rand_bits((n + pad) * batch, E, seed=9500 + 10 * E + b).reshape(batch, n + pad)
    expected = orc.oracle_permute(np.ascontiguousarray(host[:, :n]), b)
    buf = torch.from_numpy(host).to(cuda)
    rows = buf[:, :n]
    br.bitrev_batched_inplace(rows, b)
    torch.cuda.synchronize()
    assert br.last_tile() == (0, -3)
    assert_same(rows.contiguous(), expected)
    assert_same(buf[:, n:].contiguous(), np.ascontiguousarray(host[:, n:]))


@pytest.mark.parametrize("E,q", [(4, 7), (8, 6), (8, 7), (16, 5), (16, 6)])
@pytest.mark.parametrize("b,batch", [(14, 3), (15, 2), (17, 1), (20, 2), (23, 1)])
def test_cluster_pair_tiles(cuda, E, q, b, batch):
    """In-place tile pairs split over 2-CTA clusters (path 6), including the
    1 KB-row shapes the single-CTA kernel cannot hold (E=8 Q=7, E=16 Q=6),
    palindromic middles (odd and even m) and batched rows."""
    if 2 * q > b:
        pytest.skip("tile wider than the array")
    if (E, q) == (16, 6):
        pytest.skip("the default shape: below 512 MiB the size tiers route it to Q5; "
                    "covered at b = 26/27 by test_complex128_inplace_cluster_default")
    host = rand_bits(1 << b, E, seed=8000 * E + 10 * b + q, batch=batch)
    expected = orc.oracle_permute(host, b)
    old = (br.get_tile_bits(E, True), br.get_tile_path(E, True))
    try:
        br.set_tile_bits(E, True, q)
        br.set_tile_path(E, True, 6)
        a = torch.from_numpy(host).to(cuda)
        br.bitrev_batched_inplace(a, b)
        torch.cuda.synchronize()
        assert br.last_tile() == (q, 6)
        assert_same(a, expected)
    finally:
        br.set_tile_bits(E, True, old[0])
        br.set_tile_path(E, True, old[1])


@pytest.mark.parametrize("order", [0, 2])
@pytest.mark.parametrize("path", [0, 1, 2, 4, 5, 6])
@pytest.mark.parametrize("E", [4, 8, 16])
@pytest.mark.parametrize("b,batch", [(12, 2), (13, 3), (14, 3), (15, 5), (19, 2), (22, 1)])
def test_both_staging_paths(cuda, order, path, E, b, batch):
    """Register-staged and TMA-staged tile kernels, batched rows, odd and even
    widths (middle widths m = 0, 1, ... included), both families, skip-order
    and compact pair enumeration for the in-place kernels."""
    host = rand_bits(1 << b, E, seed=6000 * E + b, batch=batch)
    expected = orc.oracle_permute(host, b)
    old = (br.get_tile_path(E, False), br.get_tile_path(E, True))
    old_order = (br.get_tile_order(False), br.get_tile_order(True))
    try:
        br.set_tile_order(False, order)
        br.set_tile_order(True, order)
        br.set_tile_path(E, False, path if path < 4 else 0)
        br.set_tile_path(E, True, path)
        src = torch.from_numpy(host).to(cuda)
        out = br.bitrev_batched(src, b)
        br.bitrev_batched_inplace(src, b)
        torch.cuda.synchronize()
        assert_same(out, expected)
        assert_same(src, expected)
    finally:
        br.set_tile_path(E, False, old[0])
        br.set_tile_path(E, True, old[1])
        br.set_tile_order(False, old_order[0])
        br.set_tile_order(True, old_order[1])


@pytest.mark.parametrize("E", [4, 8, 16])
@pytest.mark.parametrize("b,batch", [(3, 5), (10, 7), (13, 3), (16, 9)])
def test_batched(cuda, E, b, batch):
    host = rand_bits(1 << b, E, seed=4000 * E + b, batch=batch)
    src = torch.from_numpy(host).to(cuda)
    out = br.bitrev_batched(src, b)
    ip = src.clone()
    br.bitrev_batched_inplace(ip, b)
    torch.cuda.synchronize()
    expected = orc.oracle_permute(host, b)
    assert_same(out, expected)
    assert_same(ip, expected)


@pytest.mark.parametrize("E", [4, 8, 16])
def test_unaligned_views_take_fallback_and_match(cuda, E):
    b = 15
    n = 1 << b
    host = rand_bits(n + 1, E, seed=5000 + E)
    base = torch.from_numpy(host).to(cuda)
    view = base[1:]  # 16-byte misaligned for E < 16... and aligned for E=16
    out = torch.empty(n + 1, dtype=base.dtype, device=cuda)[1:]
    br.cobra_out_of_place(view, out, br.CobraConfig(4), b)
    torch.cuda.synchronize()
    assert_same(out, orc.oracle_permute(host[1:], b))
    br.cobra_in_place(view, br.CobraConfig(4), b)
    torch.cuda.synchronize()
    assert_same(view, orc.oracle_permute(host[1:], b))


def test_strided_view(cuda):
    b = 12
    host = rand_bits(2 << b, 8, seed=77)
    base = torch.from_numpy(host).to(cuda)
    view = base[::2]
    expected = orc.oracle_permute(host[::2], b)
    br.xor_permute(view, b)
    torch.cuda.synchronize()
    assert_same(view, expected)
    assert_same(base[1::2], host[1::2])


def test_host_arrays_staged_through_device(cuda):
    """numpy callers of the reference API get the device path, synchronously."""
    b = 18
    host = rand_bits(1 << b, 16, seed=9)
    dest = np.empty_like(host)
    br.cobra_out_of_place(host, dest, br.CobraConfig(6), b)
    assert_same(dest, orc.oracle_permute(host, b))
    a = host.copy()
    br.recursive_permute(a, b)
    assert_same(a, orc.oracle_permute(host, b))


@pytest.mark.parametrize("b", [1, 2, 6, 11, 16, 19])
def test_involution(cuda, b):
    host = rand_bits(1 << b, 8, seed=b)
    a = torch.from_numpy(host).to(cuda)
    br.cobra_in_place(a, br.CobraConfig(0), b)
    br.cobra_in_place(a, br.CobraConfig(0), b)
    torch.cuda.synchronize()
    assert_same(a, host)


def test_canonical_vector_every_method(cuda):
    for m in br.METHOD_IDS:
        a = torch.arange(8, dtype=torch.int64, device=cuda)
        out = br.make_method(m)(a, 3)
        got = (a if out is None else out).tolist()
        assert got == [0, 4, 2, 6, 1, 5, 3, 7], m


def test_launch_counter_moves(cuda):
    before = br.launch_count()
    a = torch.arange(1 << 20, dtype=torch.float32, device=cuda)
    br.cobra_in_place(a, br.CobraConfig(6), 20)
    torch.cuda.synchronize()
    assert br.launch_count() == before + 1


@pytest.mark.parametrize("E", [4, 8, 16, 2])
@pytest.mark.parametrize("path", [0, 1, 2, 3, 4, 5, 6])
def test_guard_bands_untouched(cuda, E, path):
    """Out-of-bounds writes check (compute-sanitizer is closed on this pool):
    every staging path runs on a batched slice that sits inside a buffer with
    random guard bands before, between (row padding) and after the rows; the
    bands must come out bit-identical and the rows correct."""
    b, batch, pad = 14, 3, 4096
    n = 1 << b
    stride = n + pad  # row padding acts as an inner guard band
    buf = torch.from_numpy(rand_bits(pad + batch * stride + pad, E, seed=900 + E + 10 * path)).to(cuda)
    before = buf.clone()
    rows = buf[pad:pad + batch * stride].view(batch, stride)[:, :n]
    expected = torch.stack([br.oracle_permute(r.contiguous(), b) for r in rows])
    inplace = path != 3
    old = (br.get_tile_path(E, inplace), br.get_tile_path(E, False))
    try:
        if E in (4, 8, 16):
            br.set_tile_path(E, inplace, path if path < 4 or inplace else 0)
        if inplace:
            br.bitrev_batched_inplace(rows, b)
            got = rows
        else:
            out = torch.zeros(batch, n, dtype=buf.dtype, device=cuda)
            got = br.bitrev_batched(rows, b, out)
        torch.cuda.synchronize()
    finally:
        if E in (4, 8, 16):
            br.set_tile_path(E, inplace, old[0])
    assert_same(got, expected)
    mask = torch.ones(buf.numel(), dtype=torch.bool, device=cuda)
    if inplace:
        mask[pad:pad + batch * stride].view(batch, stride)[:, :n] = False
    assert torch.equal(buf.view(torch.uint8).view(-1, E)[mask], before.view(torch.uint8).view(-1, E)[mask])


@pytest.mark.parametrize("shape,b", [((1 << 25,), 25), ((5, 1 << 20), 20), ((3, 1 << 12), 12)])
def test_pageable_numpy_staged_copies(cuda, shape, b):
    """numpy (pageable) arrays go through the pinned bounce ring in 64 MiB
    chunks with host threads (whole, partial and single chunks), in and out of
    place, against the CPU oracle."""
    import numpy as np

    from oracle import oracle as orc

    host = np.random.default_rng(len(shape) + b).integers(0, 1 << 62, (int(np.prod(shape)) * 2,),
                                                          dtype=np.int64).view(np.complex128)
    host = host.reshape(shape)
    want = np.ascontiguousarray(orc.oracle_permute(host, b))
    dst = np.empty_like(host)
    if len(shape) == 1:
        br.cobra_out_of_place(host, dst, br.CobraConfig(6), b)
    else:
        br.bitrev_batched(host, b, dst)
    assert np.array_equal(dst.view(np.int64), want.view(np.int64))
    a = host.copy()
    if len(shape) == 1:
        br.cobra_in_place(a, br.CobraConfig(6), b)
    else:
        br.bitrev_batched_inplace(a, b)
    assert np.array_equal(a.view(np.int64), want.view(np.int64))
