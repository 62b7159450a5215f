"""Mid-size tile rule (bitrev_capi.cu small_size_q, measured by
tools/mid_sizes.py): with default knobs, launches moving at most 32 MiB per
side (64 MiB in place) use smaller tiles; one width above the budget they use
the large-size defaults; pinned knobs switch the rule off.  Every case is also
byte-compared with the oracle, so the mid-size tiles are parity-covered at the
very sizes where they run.
"""

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

NP = {4: np.int32, 8: np.int64, 16: np.complex128}
# (E, inplace) -> (mid-size q, budget MiB per side, large-size (q, path))
RULE = {(4, False): (5, 32, (7, 0)), (4, True): (5, 64, (6, 0)),
        (8, False): (4, 32, (7, 3)), (8, True): (4, 64, (6, 0)),
        (16, False): (5, 32, (6, 0)), (16, True): (5, 64, (5, 0))}


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


def budget_width(E, mib):
    return (mib << 20).bit_length() - 1 - (E.bit_length() - 1)


@pytest.mark.parametrize("E,inplace", sorted(RULE))
@pytest.mark.parametrize("above", [False, True])
def test_mid_size_rule_and_parity(cuda, E, inplace, above):
    q_mid, mib, large = RULE[(E, inplace)]
    b = budget_width(E, mib) + int(above)
    assert (E << b) == (mib << 20) << int(above)
    host = rand_bits(1 << b, E, seed=E * 100 + b)
    got, choice = run(host, b, inplace, cuda)
    assert choice == (large if above else (q_mid, 0))
    assert np.array_equal(got.view(np.uint8), orc.oracle_permute(host, b).view(np.uint8))


@pytest.mark.parametrize("E,inplace", sorted(RULE))
def test_pinned_tile_bits_disable_the_rule(cuda, E, inplace):
    _, mib, (q_large, _) = RULE[(E, inplace)]
    b = budget_width(E, mib) - 2
    q_pin = 6 if E != 16 else 4
    old = br.get_tile_bits(E, inplace)
    br.set_tile_bits(E, inplace, q_pin)
    try:
        host = rand_bits(1 << b, E, seed=E * 300 + b)
        got, (q, _) = run(host, b, inplace, cuda)
    finally:
        br.set_tile_bits(E, inplace, 0)
    assert old == q_large and q == q_pin
    assert np.array_equal(got.view(np.uint8), orc.oracle_permute(host, b).view(np.uint8))


def test_last_tile_reports_row_and_elementwise_kernels(cuda):
    x = torch.arange(1 << 10, dtype=torch.int64, device=cuda)
    br.cobra_in_place(x, br.CobraConfig(0), 10)  # 8 KB: whole-row kernel
    assert br.last_tile() == (0, -1)
    y = torch.arange(1 << 16, dtype=torch.int16, device=cuda)
    br.cobra_in_place(y, br.CobraConfig(0), 16)  # 2-byte elements: element-wise kernel
    assert br.last_tile() == (0, -2)
    torch.cuda.synchronize()
