"""CUDA-graph plans: captured launches replay to the oracle's bytes, on
refilled buffers, for every family; replay is cheaper on the host than the
eager reference-shaped call."""

import time

import pytest
import torch

import paper_1708_01873_b200 as br

pytestmark = pytest.mark.gpu


def bits(shape, dtype, cuda):
    n = 1
    for s in shape:
        n *= s
    e = torch.empty(0, dtype=dtype).element_size()
    return torch.empty(n * e, dtype=torch.uint8, device=cuda).random_(0, 256).view(dtype).view(shape)


@pytest.mark.parametrize("b,batch,dtype", [(10, 64, torch.float64), (16, 8, torch.complex128),
                                           (20, 1, torch.float32), (24, 1, torch.int64)])
def test_inplace_and_oop_plans(cuda, b, batch, dtype):
    shape = (batch, 1 << b) if batch > 1 else (1 << b,)
    x = bits(shape, dtype, cuda)
    y = torch.empty_like(x)
    p_oop = br.make_plan(x, b, y)
    p_ip = br.make_plan(x, b)
    for _ in range(2):  # refill between replays
        x.copy_(bits(shape, dtype, cuda))
        ref = torch.stack([br.oracle_permute(r, b) for r in x.view(-1, 1 << b)]).view(shape)
        p_oop.replay()
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.uint8), ref.view(torch.uint8))
        p_ip.replay()
        torch.cuda.synchronize()
        assert torch.equal(x.view(torch.uint8), ref.view(torch.uint8))


@pytest.mark.parametrize("b,batch,stages,dtype", [
    (14, 4, 7, torch.complex64),      # fused tiles
    (8, 32, 8, torch.complex64),      # short rows: complete FFT, many rows per CTA
    (13, 3, 13, torch.complex64),     # 64 KB rows: complete FFT, one row per CTA
    (10, 16, 10, torch.complex128),
])
def test_fft_plan(cuda, b, batch, stages, dtype):
    x = torch.randn(batch, 1 << b, dtype=dtype, device=cuda)
    y = torch.empty_like(x)
    plan = br.make_plan(x, b, y, stages=stages)
    plan.replay()
    torch.cuda.synchronize()
    ref = br.bitrev_dit_prepass(x, b, stages)
    assert torch.equal(y, ref)


def test_replay_cheaper_than_eager_on_host(cuda):
    b, batch = 8, 16
    x = bits((batch, 1 << b), torch.float32, cuda)
    plan = br.make_plan(x, b, replays_per_graph=1)
    for _ in range(20):
        plan.replay()
        br.bitrev_batched_inplace(x, b)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        br.bitrev_batched_inplace(x, b)
    torch.cuda.synchronize()
    eager = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(200):
        plan.replay()
    torch.cuda.synchronize()
    graph = time.perf_counter() - t0
    assert graph < eager, (graph, eager)


def test_plan_validation(cuda):
    x = torch.zeros(1 << 10, device=cuda)
    with pytest.raises(ValueError, match="overlap"):
        br.make_plan(x, 10, x)
    with pytest.raises(ValueError, match="complex"):
        br.make_plan(x, 10, torch.zeros_like(x), stages=3)
    with pytest.raises(ValueError, match="CUDA"):
        br.make_plan(torch.zeros(1 << 10), 10)


@pytest.mark.parametrize("replays", [1, 2, 3])
def test_inplace_plan_leaves_data_untouched_until_replay(cuda, replays):
    """Building an in-place plan must not permute the caller's array (its
    warm-up runs the involution twice); a replay of k launches then applies
    the permutation k times."""
    b = 18
    x = bits((1 << b,), torch.float64, cuda)
    keep = x.clone()
    plan = br.make_plan(x, b, replays_per_graph=replays)
    torch.cuda.synchronize()
    assert torch.equal(x.view(torch.uint8), keep.view(torch.uint8))
    plan.replay()
    torch.cuda.synchronize()
    want = br.oracle_permute(keep, b) if replays % 2 else keep
    assert torch.equal(x.view(torch.uint8), want.view(torch.uint8))


def test_fft_prepass_out_on_another_device_kind(cuda):
    """bitrev_dit_prepass with a CUDA input and a host (torch or numpy) or
    strided `out`: the kernel writes a device temporary that is copied back,
    never the foreign pointer."""
    import numpy as np

    b = 12
    x = bits((4, 1 << b), torch.complex64, cuda)
    want = br.bitrev_dit_prepass(x, b, 3)
    host = torch.empty(x.shape, dtype=x.dtype)
    br.bitrev_dit_prepass(x, b, 3, out=host)
    assert torch.equal(host.view(torch.uint8), want.cpu().view(torch.uint8))
    arr = np.empty((4, 1 << b), dtype=np.complex64)
    br.bitrev_dit_prepass(x, b, 3, out=arr)
    assert np.array_equal(arr.view(np.uint8), want.cpu().numpy().view(np.uint8))
    wide = torch.empty((4, 2 << b), dtype=x.dtype, device=cuda)
    view = wide[:, ::2]
    br.bitrev_dit_prepass(x, b, 3, out=view)
    assert torch.equal(view.contiguous().view(torch.uint8), want.view(torch.uint8))
