"""FFT pre-pass (bit reversal fused with radix-2 DIT stages) vs a float64
numpy restatement of the same stages, and vs np.fft for complete small FFTs.

Tolerance: complex128 |err| <= 1e-12 * max|ref|; complex64 |err| <= 2e-6 *
stages * max|ref| (float32 butterflies, twiddles rounded from float64)."""

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def dit_reference(x, b, stages, inverse=False):
    y = np.ascontiguousarray(orc.oracle_permute(x.astype(np.complex128), b))
    shape = y.shape
    for s in range(1, stages + 1):
        half = 1 << (s - 1)
        w = np.exp((2j if inverse else -2j) * np.pi * np.arange(half) / (2 * half))
        blk = y.reshape(-1, 2 * half)
        u, v = blk[:, :half], blk[:, half:] * w
        y = np.concatenate([u + v, u - v], axis=1).reshape(shape)
    return y


def check(got, ref, dtype, stages):
    got = got.cpu().numpy().astype(np.complex128)
    scale = max(np.abs(ref).max(), 1e-30)
    tol = 1e-12 if dtype == torch.complex128 else 2e-6 * max(stages, 1)
    err = np.abs(got - ref).max() / scale
    assert err <= tol, f"max rel err {err:.3e} > {tol:.1e}"


def rand_complex(shape, dtype, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    return x.astype(np.complex64 if dtype == torch.complex64 else np.complex128)


@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("b,stages", [(10, 5), (12, 6), (13, 7), (14, 6), (16, 0), (16, 3),
                                      (17, 7), (20, 6), (21, 5), (22, 7)])
@pytest.mark.parametrize("inverse", [False, True])
def test_fused_stages_match_reference(cuda, dtype, b, stages, inverse):
    if dtype == torch.complex128 and stages > 6 and (1 << b) * 16 > 32768:
        pytest.skip("complex128 tiles fuse at most 6 stages")
    x = rand_complex(1 << b, dtype, b * 10 + stages)
    got = br.bitrev_dit_prepass(torch.from_numpy(x).to(cuda), b, stages, inverse=inverse)
    check(got, dit_reference(x, b, stages, inverse), dtype, stages)


@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
@pytest.mark.parametrize("b", [1, 2, 5, 8, 11, 12, 13])
def test_small_rows_full_fft(cuda, dtype, b):
    """Rows up to 64 KB take any number of stages: a complete FFT."""
    if (1 << b) * (8 if dtype == torch.complex64 else 16) > 65536:
        pytest.skip("row too long for a complete fused FFT")
    x = rand_complex((3, 1 << b), dtype, b)
    got = br.bitrev_dit_prepass(torch.from_numpy(x).to(cuda), b, b)
    check(got, np.fft.fft(x.astype(np.complex128), axis=-1), dtype, b)
    inv = br.bitrev_dit_prepass(torch.from_numpy(x).to(cuda), b, b, inverse=True)
    check(inv, np.fft.ifft(x.astype(np.complex128), axis=-1) * (1 << b), dtype, b)


def test_zero_stages_is_the_permutation(cuda):
    b = 18
    x = torch.from_numpy(rand_complex(1 << b, torch.complex64, 1)).to(cuda)
    got = br.bitrev_dit_prepass(x, b, 0)
    assert torch.equal(got.view(torch.int64), br.oracle_permute(x, b).view(torch.int64))


def test_batched_and_host_arrays(cuda):
    b, stages = 16, 6
    x = rand_complex((5, 1 << b), torch.complex128, 7)
    got = br.bitrev_dit_prepass(x, b, stages)  # numpy in -> staged through the device
    check(got, dit_reference(x, b, stages), torch.complex128, stages)


@pytest.mark.parametrize("dtype,fused", [(torch.complex128, 6), (torch.complex64, 7)])
def test_completes_to_torch_fft(cuda, dtype, fused):
    """prepass (fused stages) + the remaining DIT stages in torch == torch.fft.fft."""
    b = 16
    x = torch.from_numpy(rand_complex(1 << b, dtype, 3)).to(cuda).to(torch.complex128)
    y = br.bitrev_dit_prepass(x.to(dtype), b, fused).to(torch.complex128)
    for s in range(fused + 1, b + 1):
        half = 1 << (s - 1)
        w = torch.exp(-2j * torch.pi * torch.arange(half, device=cuda, dtype=torch.float64)
                      / (2 * half))
        blk = y.view(-1, 2 * half)
        u, v = blk[:, :half], blk[:, half:] * w
        y = torch.cat([u + v, u - v], dim=1).reshape(-1)
    ref = torch.fft.fft(x)
    tol = 1e-9 if dtype == torch.complex128 else 1e-5
    assert (y - ref).abs().max().item() <= tol * ref.abs().max().item()


def test_validation(cuda):
    x = torch.zeros(1 << 14, dtype=torch.float32, device=cuda)
    with pytest.raises(ValueError, match="complex"):
        br.bitrev_dit_prepass(x, 14, 2)
    z = torch.zeros(1 << 14, dtype=torch.complex64, device=cuda)
    with pytest.raises(ValueError, match="stages"):
        br.bitrev_dit_prepass(z, 14, 15)
    with pytest.raises(br.BitrevError):
        br.bitrev_dit_prepass(z, 14, 9)  # complex64 tiles fuse at most 7 stages
    assert br.max_fused_stages(14, 8) == 7 and br.max_fused_stages(14, 16) == 6
    assert br.max_fused_stages(11, 16) == 11


@pytest.mark.parametrize("stages", [2, 5, 7])
def test_cfg4_shape_batched_complex64(cuda, stages):
    """cfg4's shape (rows of 2^16 complex64, here 16 of them) through the
    256-byte-piece tiles (2-6 stages) and the radix-8 drain (7 stages), forward
    and inverse, every row against the float64 restatement."""
    b = 16
    x = rand_complex((16, 1 << b), torch.complex64, 40 + stages)
    for inverse in (False, True):
        got = br.bitrev_dit_prepass(torch.from_numpy(x).to(cuda), b, stages, inverse=inverse)
        ref = np.stack([dit_reference(r, b, stages, inverse) for r in x])
        check(got, ref, torch.complex64, stages)


@pytest.mark.parametrize("b,rows,stages", [(16, 80, 1), (16, 80, 2), (16, 80, 3), (16, 80, 4),
                                           (16, 80, 5), (16, 80, 6), (14, 128, 6), (14, 128, 7),
                                           (13, 256, 7), (22, 1, 3)])
def test_wide_rows_tier_complex64(cuda, b, rows, stages):
    """complex64 launches of >= 16 MiB take the 256-element destination rows
    (two FFT blocks per row, radix-8 drain: bitrev_dit_prepass's QX = 8 rule)
    for 1-5 stages, and for 6-7 stages on rows of 2^13-2^14; the other 6-7
    stage cases stay on 128-element rows.  Forward and inverse, every row
    against the float64 restatement."""
    x = rand_complex((rows, 1 << b), torch.complex64, 70 + stages + b)
    for inverse in (False, True):
        got = br.bitrev_dit_prepass(torch.from_numpy(x).to(cuda), b, stages, inverse=inverse)
        ref = np.stack([dit_reference(r, b, stages, inverse) for r in x])
        check(got, ref, torch.complex64, stages)


@pytest.mark.parametrize("stages,pinned", [(7, True), (3, True), (5, False)])
def test_dit_prepass_host_pipeline(cuda, stages, pinned):
    """dit_prepass_host_pipeline over host arrays (pinned: overlapped copies;
    numpy/pageable: the bounce-ring path), out of place and over the inputs,
    a recurring array included: every result equals the device call's bytes."""
    b, rows = 16, 24
    xs = [rand_complex((rows, 1 << b), torch.complex64, 90 + k) for k in range(4)]
    want = [br.bitrev_dit_prepass(torch.from_numpy(x).to(cuda), b, stages).cpu() for x in xs]
    if pinned:
        hs = [torch.from_numpy(x).pin_memory() for x in xs]
        outs = [torch.empty_like(h).pin_memory() for h in hs]
    else:
        hs = [x.copy() for x in xs]
        outs = [np.empty_like(x) for x in xs]
    seq_in = hs + [hs[0]]
    seq_out = outs + [outs[0]]
    got = br.dit_prepass_host_pipeline(seq_in, b, stages, out=seq_out)
    for k in range(4):
        g = torch.as_tensor(got[k])
        assert torch.equal(g.view(torch.uint8), want[k].view(torch.uint8)), k
    # in place on the host (out=None): each input replaced by its result
    ins = [h.clone() if pinned else h.copy() for h in hs]
    if pinned:
        ins = [t.pin_memory() for t in ins]
    br.dit_prepass_host_pipeline(ins, b, stages)
    for k in range(4):
        assert torch.equal(torch.as_tensor(ins[k]).view(torch.uint8), want[k].view(torch.uint8))


def test_dit_prepass_host_pipeline_validation(cuda):
    x = torch.zeros(1 << 10, dtype=torch.complex64)
    with pytest.raises(ValueError, match="complex"):
        br.dit_prepass_host_pipeline([torch.zeros(1 << 10)], 10, 2)
    with pytest.raises(ValueError, match="stages"):
        br.dit_prepass_host_pipeline([x], 10, 11)
    with pytest.raises(ValueError, match="host arrays"):
        br.dit_prepass_host_pipeline([x.to(cuda)], 10, 2)
    with pytest.raises(ValueError, match="one destination"):
        br.dit_prepass_host_pipeline([x, x.clone()], 10, 2, out=[x.clone()])
    assert br.dit_prepass_host_pipeline([], 10, 2) == []


@pytest.mark.parametrize("b,rows", [(12, 16), (14, 4), (18, 1)])
@pytest.mark.parametrize("stages", [1, 2, 3, 4, 5])
def test_complex128_square_tiles_shuffle_stages(cuda, b, rows, stages):
    """complex128 with 1-5 stages on rows of 2^12 and up: the square Q6 tiles
    with the butterflies on warp shuffles (bitrev_fft_tile16_kernel), forward
    and inverse, every row against the float64 restatement."""
    x = rand_complex((rows, 1 << b), torch.complex128, 200 + 10 * b + stages)
    for inverse in (False, True):
        got = br.bitrev_dit_prepass(torch.from_numpy(x).to(cuda), b, stages, inverse=inverse)
        ref = np.stack([dit_reference(r, b, stages, inverse) for r in x])
        check(got, ref, torch.complex128, stages)


@pytest.mark.parametrize("dtype,b,rows,stages", [
    (torch.complex64, 16, 80, 3),    # 256-element rows (>= 16 MiB)
    (torch.complex64, 16, 8, 7),     # 128-element rows, radix-8 drain
    (torch.complex128, 14, 8, 2),    # square tiles, shuffle stages
    (torch.complex128, 14, 8, 6),    # rectangular tiles, radix-4 drain
])
def test_strided_rows_through_the_c_abi(cuda, dtype, b, rows, stages):
    """bitrev_dit_prepass with batch strides wider than the rows (rows inside
    padded buffers): results equal the contiguous call's bytes and the pads
    on both sides stay untouched."""
    from paper_1708_01873_b200 import _core, _lib

    n, sp, dp = 1 << b, 24, 40
    E = 8 if dtype == torch.complex64 else 16
    x = torch.from_numpy(rand_complex((rows, n), dtype, 300 + b + stages)).to(cuda)
    src = torch.full((rows, n + sp), complex(7.0, -7.0), dtype=dtype, device=cuda)
    src[:, :n] = x
    dst = torch.full((rows, n + dp), complex(3.0, 5.0), dtype=dtype, device=cuda)
    _lib.call("bitrev_dit_prepass", src.data_ptr(), dst.data_ptr(), b, E, rows, n + sp, n + dp,
              stages, 0, _core._stream_ptr(x.device))
    want = br.bitrev_dit_prepass(x, b, stages)
    torch.cuda.synchronize()
    assert torch.equal(dst[:, :n].view(torch.uint8), want.view(torch.uint8))
    assert bool((dst[:, n:] == complex(3.0, 5.0)).all())
    assert bool((src[:, n:] == complex(7.0, -7.0)).all())
