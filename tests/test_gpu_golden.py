"""GPU parity against the reference's golden vectors and size-independent
properties at the BASELINE sizes.

* every golden case (tests/golden/golden.json, produced by running the
  reference package) x every method id through make_method on CUDA tensors:
  SHA-256 of the output bytes must equal the reference's;
* the acceptance criteria of the reference (canonical vector, involution,
  transposition, even-odd) on the device;
* at b = 26..30 (BASELINE configs 2/3) where the CPU oracle is slow: sentinel
  self-check (value = index => out[i] == rev(i), computed by an independent
  torch shift loop) and a sampled CPU-oracle check;
* the sharded plan's kernels through emulate_sharded vs the oracle.
"""

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from oracle import oracle as orc
from paper_1708_01873_b200 import sharded

pytestmark = pytest.mark.gpu

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())
sys.path.insert(0, str(Path(__file__).parent / "golden"))
from recipes import make_input  # noqa: E402


def sha_t(t):
    a = t.detach().cpu().contiguous().numpy()
    return hashlib.sha256(a.view(np.uint8).tobytes()).hexdigest()


def case_id(c):
    return f"{c['recipe']}-E{c['E']}-b{c['b']}-t{c['trial']}"


@pytest.mark.parametrize("c", GOLDEN["cases"], ids=case_id)
def test_every_method_matches_reference_digest(cuda, c):
    x = make_input(c["recipe"], c["E"], c["b"], c["trial"])
    src = torch.from_numpy(x).to(cuda)
    for m in br.METHOD_IDS:
        a = src.clone()
        out = br.make_method(m)(a, c["b"])
        got = a if out is None else out
        assert sha_t(got) == c["output_sha256"], m
    # oracle_permute (independent torch gather) and the batched entry point
    assert sha_t(br.oracle_permute(src, c["b"])) == c["output_sha256"]
    assert sha_t(br.bitrev_batched(src.view(1, -1), c["b"])) == c["output_sha256"]


def test_canonical_and_acceptance_small(cuda):
    for m, want in GOLDEN["canonical"].items():
        a = torch.arange(8, dtype=torch.int64, device=cuda)
        out = br.make_method(m)(a, 3)
        assert (a if out is None else out).tolist() == want
    for b, table in GOLDEN["rev_index_small"].items():
        assert br.rev_index_array(int(b), cuda).tolist() == table


def test_transpose_square_golden(cuda):
    for h, case in GOLDEN["transpose_square"].items():
        t = torch.tensor(case["input"], dtype=torch.int64, device=cuda)
        br.transpose_square_inplace(t, int(h))
        assert t.tolist() == case["output"]
    for h in (5, 6, 9, 10):
        x = torch.randint(0, 1 << 30, (1 << (2 * h),), device=cuda, dtype=torch.int64)
        w = x.clone()
        br.transpose_square_inplace(w, h)
        side = 1 << h
        assert torch.equal(w, x.view(side, side).t().reshape(-1))
        br.transpose_square_inplace(w, h)
        assert torch.equal(w, x)


def test_even_odd_golden(cuda):
    t = torch.arange(16, dtype=torch.int64, device=cuda)
    br.even_odd_permute(t, 4)
    assert t.tolist() == GOLDEN["even_odd_b4"]
    x = torch.randint(0, 1 << 30, (1 << 20,), device=cuda, dtype=torch.int32)
    w = x.clone()
    br.even_odd_permute(w, 20)
    assert torch.equal(w, torch.cat([x[0::2], x[1::2]]))


def test_explicit_pair_schedule(cuda):
    b = 12
    r = orc.rev_index_array(b)
    i = np.arange(1 << b)
    pairs = np.stack([i[i < r], r[i < r]], axis=1)
    x = torch.randint(0, 1 << 30, (1 << b,), device=cuda, dtype=torch.int64)
    a = x.clone()
    br.apply_schedule(a, br.SwapSchedule(b, pairs))
    assert torch.equal(a, br.oracle_permute(x, b))
    a = x.clone()
    br.apply_schedule(a, br.cached_schedule(b))
    assert torch.equal(a, br.oracle_permute(x, b))


def _torch_rev(b, dev):
    idx = torch.arange(1 << b, dtype=torch.int64, device=dev)
    out = torch.zeros_like(idx)
    for _ in range(b):
        out = (out << 1) | (idx & 1)
        idx >>= 1
    return out


@pytest.mark.parametrize("b,dtype,inplace", [
    (26, torch.int64, True),    # config 2 (float64 bit width)
    (26, torch.int64, False),
    (28, torch.int32, False),
    (28, torch.int32, True),
    (30, torch.int32, False),   # config 3, E = 4
    (30, torch.int32, True),
])
def test_sentinel_self_check_large(cuda, b, dtype, inplace):
    a = torch.arange(1 << b, dtype=dtype, device=cuda)
    if inplace:
        br.cobra_in_place(a, br.CobraConfig(6), b)
        out = a
    else:
        out = torch.empty_like(a)
        br.cobra_out_of_place(a, out, br.CobraConfig(6), b)
    expect = _torch_rev(b, cuda).to(dtype)
    assert torch.equal(out, expect)


@pytest.mark.parametrize("b", [28, 29])
def test_complex128_large_sampled_vs_cpu_oracle(cuda, b):
    """E = 16 at large b: random bits on device, the permutation checked at
    2^20 random positions against the CPU rev_naive (and involution)."""
    n = 1 << b
    x = torch.empty(n * 16, dtype=torch.uint8, device=cuda)
    x.random_(0, 256)
    x = x.view(torch.complex128)
    out = torch.empty_like(x)
    br.cobra_out_of_place(x, out, br.CobraConfig(6), b)
    idx = np.random.default_rng(b).integers(0, n, 1 << 20)
    ridx = orc.rev_index_array(b)[idx] if b <= 28 else np.array([orc.rev_naive(int(i), b)
                                                                  for i in idx[:4096]])
    idx = idx[: len(ridx)]
    xi = x.view(torch.int64).view(-1, 2)
    oi = out.view(torch.int64).view(-1, 2)
    ti = torch.from_numpy(idx).to(cuda)
    tr = torch.from_numpy(np.asarray(ridx)).to(cuda)
    assert torch.equal(oi[ti], xi[tr])
    br.cobra_in_place(out, br.CobraConfig(6), b)
    assert torch.equal(out.view(torch.int64), x.view(torch.int64))


@pytest.mark.parametrize("b,batch", [(26, 1), (26, 2), (27, 1)])
def test_complex128_inplace_cluster_default(cuda, b, batch):
    """complex128 in place above the mid-size tier runs the 2-CTA cluster pair
    kernel by default (even and odd middle widths, batched rows); every byte
    is compared with the device oracle."""
    x = torch.empty(batch * (1 << b) * 16, dtype=torch.uint8, device=cuda).random_(0, 256)
    x = x.view(torch.complex128).view(batch, 1 << b)
    expect = torch.stack([br.oracle_permute(r, b) for r in x])
    br.bitrev_batched_inplace(x, b)
    torch.cuda.synchronize()
    assert br.last_tile() == (6, 6)
    assert torch.equal(x.view(torch.uint8), expect.view(torch.uint8))


@pytest.mark.parametrize("b,G,dtype,chunks", [(12, 2, torch.int64, 1), (16, 4, torch.complex64, 1),
                                              (20, 8, torch.float32, 4), (21, 8, torch.complex128, 2),
                                              (26, 8, torch.complex64, 8), (14, 2, torch.int32, 16)])
def test_sharded_plan_kernels(cuda, b, G, dtype, chunks):
    x = torch.empty((1 << b) * torch.empty(0, dtype=dtype).element_size(), dtype=torch.uint8,
                    device=cuda).random_(0, 256).view(dtype)
    outs = sharded.emulate_sharded(x, b, G, chunks)
    got = torch.cat(outs)
    assert torch.equal(got.view(torch.uint8), br.oracle_permute(x, b).view(torch.uint8))


def _chunked_rev_check(out, b, chunk_bits=27):
    """out[i] == rev_b(i) for every i, verified 2^chunk_bits indices at a time
    with an independent torch shift loop (keeps the check's memory bounded)."""
    dev = out.device
    n = 1 << b
    for start in range(0, n, 1 << chunk_bits):
        idx = torch.arange(start, min(n, start + (1 << chunk_bits)), dtype=torch.int64, device=dev)
        r = torch.zeros_like(idx)
        v = idx.clone()
        for _ in range(b):
            r = (r << 1) | (v & 1)
            v >>= 1
        assert torch.equal(out[start:start + idx.numel()].to(torch.int64), r), start


@pytest.mark.parametrize("b,inplace", [(31, True), (31, False), (32, True)])
def test_sentinel_64bit_sizes(cuda, b, inplace):
    """2^31 / 2^32 int64 elements (16 / 32 GiB): the sizes of BASELINE config
    5's shards and beyond; exercises 64-bit offsets in every index path."""
    free, _ = torch.cuda.mem_get_info(cuda)
    need = (1 << b) * 8 * (1 if inplace else 2) + (6 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB free")
    a = torch.arange(1 << b, dtype=torch.int64, device=cuda)
    if inplace:
        br.cobra_in_place(a, br.CobraConfig(6), b)
        out = a
    else:
        out = torch.empty_like(a)
        br.cobra_out_of_place(a, out, br.CobraConfig(6), b)
        del a
    torch.cuda.synchronize()
    _chunked_rev_check(out, b)


@pytest.mark.parametrize("b,G,dtype", [(16, 2, torch.int64), (18, 4, torch.float32),
                                       (20, 8, torch.complex128), (26, 8, torch.complex64),
                                       (24, 8, torch.int32), (14, 2, torch.int32)])
def test_sharded_p2p_scatter_kernel(cuda, b, G, dtype):
    """Fused local-reversal + scatter into the peers' receive buffers
    (bitrev_sharded_scatter: rectangular tiles, or square tiles for a shard
    narrower than a rectangular tile, b = 14 float32), all ranks emulated on
    one device."""
    x = torch.empty((1 << b) * torch.empty(0, dtype=dtype).element_size(), dtype=torch.uint8,
                    device=cuda).random_(0, 256).view(dtype)
    got = torch.cat(sharded.emulate_sharded_p2p(x, b, G))
    assert torch.equal(got.view(torch.uint8), br.oracle_permute(x, b).view(torch.uint8))


@pytest.mark.parametrize("c", [c for c in GOLDEN["cases"] if c["b"] in (5, 12, 17) and
                               c["recipe"] == "bits"], ids=case_id)
def test_numpy_callers_get_reference_bytes(cuda, c):
    """Drop-in: every method id driven with NUMPY arrays (the reference's own
    array type) is staged through the device and matches the reference digest;
    out-of-place results come back as numpy arrays."""
    x = make_input(c["recipe"], c["E"], c["b"], c["trial"])
    for m in br.METHOD_IDS:
        a = x.copy()
        out = br.make_method(m)(a, c["b"])
        got = a if out is None else out
        assert isinstance(got, np.ndarray), m
        assert hashlib.sha256(np.ascontiguousarray(got).view(np.uint8).tobytes()).hexdigest() \
            == c["output_sha256"], m
    o = br.oracle_permute(x, c["b"])
    assert isinstance(o, np.ndarray)
    assert hashlib.sha256(o.view(np.uint8).tobytes()).hexdigest() == c["output_sha256"]
