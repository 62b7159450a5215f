"""Mid-size tile tiers (bitrev_capi.cu mid_tier, measured by
tools/mid_sizes.py): with default knobs, launches below per-family byte
budgets use smaller tiles, and one width above the last budget the large-size
defaults; a non-default knob value switches the tiers off.  Every case is
also byte-compared with the oracle, so the mid-size tiles are parity-covered
at the very sizes where they run.
"""

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

NP = {4: np.int32, 8: np.int64, 16: np.complex128}
# (E, inplace) -> default (q, path) above every budget
LARGE = {(4, False): (8, 3), (4, True): (6, 0), (8, False): (7, 3), (8, True): (6, 0),
         (16, False): (6, 0), (16, True): (6, 6)}
# (E, inplace, b, expected (q, path)) at each budget and one width above it
CASES = [
    (4, False, 23, (5, 0)), (4, False, 24, (7, 3)),    # 32 MiB tier: square Q5
    (4, False, 25, (8, 3)),                            # above the 64 MiB rect QX=7 tier
    (4, True, 24, (5, 0)), (4, True, 25, (6, 0)),
    (8, False, 22, (4, 0)), (8, False, 23, (7, 3)),
    (8, True, 23, (4, 0)), (8, True, 24, (6, 0)),
    (16, False, 19, (5, 0)), (16, False, 20, (4, 2)),    # 8 MiB: register Q5; 32 MiB: TMA ring Q4
    (16, False, 21, (4, 2)), (16, False, 22, (6, 0)),
    (16, True, 25, (5, 0)), (16, True, 26, (6, 6)),    # 512 MiB tier: single-CTA pairs
]
# pinned values that differ from the default and from any tier's q
PIN = {(4, False): 6, (4, True): 7, (8, False): 6, (8, True): 5, (16, False): 4, (16, True): 4}


def rand_bits(n, E, seed):
    raw = np.random.default_rng(seed).integers(0, 256, size=n * E, dtype=np.uint8)
    return raw.view(NP[E])


def run(host, b, inplace, cuda):
    src = torch.from_numpy(host).to(cuda)
    if inplace:
        br.cobra_in_place(src, br.CobraConfig(0), b)
        out = src
    else:
        out = torch.empty_like(src)
        br.cobra_out_of_place(src, out, br.CobraConfig(0), b)
    torch.cuda.synchronize()
    return out.cpu().numpy(), br.last_tile()


@pytest.mark.parametrize("E,inplace,b,expected", CASES)
def test_mid_size_tiers_and_parity(cuda, E, inplace, b, expected):
    host = rand_bits(1 << b, E, seed=E * 100 + b)
    got, choice = run(host, b, inplace, cuda)
    assert choice == expected
    assert np.array_equal(got.view(np.uint8), orc.oracle_permute(host, b).view(np.uint8))


@pytest.mark.parametrize("E,inplace", sorted(LARGE))
def test_pinned_tile_bits_disable_the_tiers(cuda, E, inplace):
    """Tile bits set to a non-default value switch the tiers off; setting the
    default value back (save/restore) switches them on again."""
    b = 20
    old = br.get_tile_bits(E, inplace)
    assert old == LARGE[(E, inplace)][0]
    br.set_tile_bits(E, inplace, PIN[(E, inplace)])
    try:
        host = rand_bits(1 << b, E, seed=E * 300 + b)
        got, (q, _) = run(host, b, inplace, cuda)
    finally:
        br.set_tile_bits(E, inplace, old)  # by value: the default again
    assert q == PIN[(E, inplace)]
    assert np.array_equal(got.view(np.uint8), orc.oracle_permute(host, b).view(np.uint8))
    _, choice = run(host, b, inplace, cuda)
    at20 = [c[3] for c in CASES if c[:3] == (E, inplace, 20)]
    small = min((c for c in CASES if c[:2] == (E, inplace)), key=lambda c: c[2])
    assert choice == (at20[0] if at20 else small[3])  # b=20's tier again


def test_last_tile_reports_row_and_elementwise_kernels(cuda):
    x = torch.arange(1 << 10, dtype=torch.int64, device=cuda)
    br.cobra_in_place(x, br.CobraConfig(0), 10)  # 8 KB aligned rows: short-row kernel
    assert br.last_tile() == (0, -3)
    h = torch.arange(1 << 10, dtype=torch.int16, device=cuda)
    br.cobra_in_place(h, br.CobraConfig(0), 10)  # 2-byte elements, 2 KB: whole-row kernel
    assert br.last_tile() == (0, -1)
    y = torch.arange(1 << 16, dtype=torch.int16, device=cuda)
    br.cobra_in_place(y, br.CobraConfig(0), 16)  # 2-byte elements: element-wise kernel
    assert br.last_tile() == (0, -2)
    torch.cuda.synchronize()


# batched 8-byte rows out of place (bitrev_capi.cu batched_rows_tier): rows of
# 2^13..2^22 elements past the 32 MiB budget take 2 KB destination rows
BATCHED = [
    (13, 8192, (8, 3)), (16, 64, (4, 0)), (16, 128, (8, 3)), (22, 2, (8, 3)),
    (23, 2, (7, 3)),       # rows above 2^22: the default
    (12, 16384, (0, -3)),  # 32 KB rows: the short-row kernel
]


@pytest.mark.parametrize("b,rows,expected", BATCHED)
def test_batched_rows_tier_and_parity(cuda, b, rows, expected):
    x = torch.empty((rows, 1 << b), dtype=torch.float64, device=cuda).normal_()
    x.view(torch.int64)[:, :7] = torch.tensor([0x7FF8000000000001, -1, 0, -(1 << 63), 1, 2, 3])
    out = br.bitrev_batched(x, b)
    torch.cuda.synchronize()
    assert br.last_tile() == expected
    idx = torch.from_numpy(orc.rev_index_array(b)).to(cuda)
    assert torch.equal(out.view(torch.int64), x.view(torch.int64).index_select(1, idx))


def test_batched_rows_tier_off_with_pinned_knobs(cuda):
    old = br.get_tile_bits(8, False)
    br.set_tile_bits(8, False, 6)
    try:
        x = torch.empty((128, 1 << 16), dtype=torch.float64, device=cuda).normal_()
        br.bitrev_batched(x, 16)
        assert br.last_tile()[0] == 6
    finally:
        br.set_tile_bits(8, False, old)
    br.bitrev_batched(x, 16)
    assert br.last_tile() == (8, 3)
