"""The index maths the tile kernels rely on, restated in Python (CPU).

* the tile identity rev_b(x*2^(b-Q) + y*2^Q + z) = rev_Q(z)*2^(b-Q) +
  rev_m(y)*2^Q + rev_Q(x) (csrc/bitrev_kernels.cuh header);
* the register transpose row trick rev_Q(g + k*2^Q/V) = rev_{Q-LV}(g)*V +
  rev_LV(k);
* work_to_y (tile visit orders) is a bijection for every code;
* pair_from_index enumerates exactly the canonical pairs {y <= rev(y)},
  and pair_count matches the swap-count law (src/schedule.py:23-37) plus
  palindromes.
The CUDA versions are exercised byte-exactly by the GPU parity tests.
"""

import pytest

from oracle.oracle import rev_naive as rev


def rev0(v, w):
    return rev(v, w) if w else 0


def work_to_y(w, m, order):
    if order == 0 or m < 2:
        return w
    if order == 1:
        h = m >> 1
        even = [(w >> (2 * k)) & 1 for k in range(h)]
        odd = [(w >> (2 * k + 1)) & 1 for k in range(h)]
        y = sum(bit << k for k, bit in enumerate(even))
        y |= sum(bit << (m - 1 - k) for k, bit in enumerate(odd))
        if m & 1:
            y |= ((w >> (2 * h)) & 1) << h
        return y
    L, H = (order >> 4) & 15, order & 15
    L = min(L, m)
    H = min(H, m - L)
    lo = w & ((1 << L) - 1)
    hi = (w >> L) & ((1 << H) - 1)
    mid = w >> (L + H)
    return (hi << (m - H)) | (mid << L) | lo


def pair_count(m):
    return ((1 << m) + (1 << ((m + 1) // 2))) >> 1


def pair_from_index(w, m):
    if m == 0:
        return 0
    h = m >> 1
    Sh = (1 << (m - 1)) - (1 << (m - h - 1))
    if w < Sh:
        k = 0
        while (w >> (m - 2 - k)) & 1:
            k += 1
        o = w - ((1 << (m - 1)) - (1 << (m - k - 1)))
        ib = m - 2 * k - 2
        inner, outer = o & ((1 << ib) - 1), o >> ib
        return (inner << (k + 1)) | (1 << k) | outer | (rev0(outer, k) << (m - k))
    p = w - Sh
    outer = p & ((1 << h) - 1)
    y = outer | (rev0(outer, h) << (m - h))
    if m & 1:
        y |= ((p >> h) & 1) << h
    return y


@pytest.mark.parametrize("b,Q", [(6, 3), (7, 3), (10, 4), (11, 5), (12, 6)])
def test_tile_identity(b, Q):
    m = b - 2 * Q
    for i in range(1 << b):
        x, y, z = i >> (b - Q), (i >> Q) & ((1 << m) - 1), i & ((1 << Q) - 1)
        assert rev(i, b) == (rev(z, Q) << (b - Q)) | (rev0(y, m) << Q) | rev(x, Q)


@pytest.mark.parametrize("Q,V", [(5, 1), (5, 2), (5, 4), (6, 2), (6, 4), (7, 4)])
def test_register_transpose_rows(Q, V):
    LV = V.bit_length() - 1
    G = (1 << Q) // V
    for g in range(G):
        for k in range(V):
            assert rev(g + k * G, Q) == rev0(g, Q - LV) * V + rev0(k, LV)


@pytest.mark.parametrize("order", [0, 1, 0x160, 0x183, 0x1A4, 0x1F6])
@pytest.mark.parametrize("m", range(0, 13))
def test_work_to_y_bijection(order, m):
    assert sorted(work_to_y(w, m, order) for w in range(1 << m)) == list(range(1 << m))


@pytest.mark.parametrize("m", range(0, 15))
def test_pair_enumeration(m):
    canon = sorted(y for y in range(1 << m) if rev0(y, m) >= y)
    ys = [pair_from_index(w, m) for w in range(pair_count(m))]
    assert sorted(ys) == canon
    if m >= 1:
        swaps = ((1 << m) - (1 << ((m + 1) // 2))) // 2  # src/schedule.py:23-37 closed form
        assert pair_count(m) == swaps + (1 << ((m + 1) // 2))
