"""Dedicated kernels of the remaining entry points.

* transpose_square_inplace: the vectorised tile-pair transpose (h >= 5/6 for
  4/8/16-byte elements, aligned) and the scalar kernel (1/2-byte elements,
  small h), every element against torch's .t(), batched through the C ABI;
* even_odd_permute: the two in-place bit reversals it factors into, against
  the definition new[j] = old[2j], new[n/2 + j] = old[2j + 1] (the reference's
  _even_odd, src/recursive.py:84-93), for every element width, device and
  host arrays, strided views.
"""

import ctypes

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from paper_1708_01873_b200 import _lib

pytestmark = pytest.mark.gpu

DTYPES = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64, 16: torch.complex128}


def rand(n, E, dev):
    return torch.empty(n * E, dtype=torch.uint8, device=dev).random_(0, 256).view(DTYPES[E])


@pytest.mark.parametrize("E", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("h", [1, 3, 5, 6, 7, 10, 12])
def test_transpose_every_width(cuda, E, h):
    x = rand(1 << (2 * h), E, cuda)
    w = x.clone()
    br.transpose_square_inplace(w, h)
    side = 1 << h
    assert torch.equal(w.view(torch.uint8), x.view(side, side).t().contiguous().view(-1).view(torch.uint8))


@pytest.mark.parametrize("E,h", [(4, 7), (8, 6), (16, 5), (2, 6)])
def test_transpose_batched_capi(cuda, E, h):
    n, batch = 1 << (2 * h), 3
    stride = n + (64 // E)  # padded rows, still 16-byte aligned
    buf = rand(batch * stride, E, cuda)
    keep = buf.clone()
    _lib.call("bitrev_transpose_square", buf.data_ptr(), h, E, batch, stride,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    side = 1 << h
    for k in range(batch):
        want = keep[k * stride:k * stride + n].view(side, side).t().contiguous().view(-1)
        assert torch.equal(buf[k * stride:k * stride + n].view(torch.uint8), want.view(torch.uint8))
        assert torch.equal(buf[k * stride + n:(k + 1) * stride].view(torch.uint8),
                           keep[k * stride + n:(k + 1) * stride].view(torch.uint8))


def even_odd_ref(x):
    return torch.cat([x[0::2], x[1::2]])


@pytest.mark.parametrize("E", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("b", [1, 2, 3, 7, 12, 17, 22])
def test_even_odd_every_width(cuda, E, b):
    x = rand(1 << b, E, cuda)
    w = x.clone()
    br.even_odd_permute(w, b)
    assert torch.equal(w.view(torch.uint8), even_odd_ref(x).view(torch.uint8))


def test_even_odd_host_and_strided(cuda):
    b = 14
    host = np.random.default_rng(1).integers(0, 1 << 40, 1 << b)
    want = np.concatenate([host[0::2], host[1::2]])
    h = host.copy()
    br.even_odd_permute(h, b, scratch=np.empty(1 << (b - 1), dtype=h.dtype))
    assert np.array_equal(h, want)
    big = torch.from_numpy(np.stack([host, host], 1).reshape(-1)).to(cuda)
    view = big[0::2]  # strided device view
    br.even_odd_permute(view, b)
    assert np.array_equal(view.cpu().numpy(), want)
    assert np.array_equal(big[1::2].cpu().numpy(), host)  # the other lane untouched
