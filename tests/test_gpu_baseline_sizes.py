"""Every-element parity at the BASELINE.json sizes.

The reference's own acceptance protocol compares every method's output with
oracle_permute element by element (/root/reference/pkg/tests/test_acceptance.py:
42-70).  At the BASELINE sizes the CPU oracle is too slow (and at 2^30
complex128 too big for a comfortable host copy), so the same comparison runs
on the device, chunk by chunk, against an oracle that shares no code with the
kernels: the reversed index of every output slot is rebuilt with a torch shift
loop (one pass per bit, like rev_index_array, src/verify.py:19-31) and the
source is gathered through it with index_select.  Comparisons are on raw
words (int32 / int64 views), so NaN payloads and -0.0 are bytes like any other.

* config 3: 2^30 float32 / float64 / complex128 out of place, random bit
  patterns, every element; then the in-place path on the same array must
  reproduce the out-of-place bytes;
* config 3, complex128: the (i, ~i) u64 sentinel pairs of SURVEY 8(c5), every
  element;
* config 2: 2^26 float64 in place with a float64 payload (normals, NaNs with
  payload bits, signed zeros, infinities) against the CPU oracle;
* config 4: the full 4096 x 2^16 complex64 batch against the CPU oracle;
* config 5's plan at 2^31 complex64 over 8 emulated ranks (16 GiB), every
  element, with the sub-chunked exchange layout; and at config 5's own size,
  2^32 complex64 (32 GiB) over 2 / 4 / 8 emulated ranks (pack + rounds +
  unpack) and 8 ranks of the fused peer-store scatter.
"""

import gc

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from oracle import oracle as orc
from paper_1708_01873_b200 import sharded, verify

pytestmark = pytest.mark.gpu

CHUNK_BITS = 26


@pytest.fixture(autouse=True)
def _free_device_memory():
    verify._REV_CACHE.clear()
    gc.collect()
    torch.cuda.empty_cache()
    yield
    verify._REV_CACHE.clear()
    gc.collect()
    torch.cuda.empty_cache()


def _need(cuda, nbytes):
    free, _ = torch.cuda.mem_get_info(cuda)
    if free < nbytes + (4 << 30):
        pytest.skip(f"needs {(nbytes >> 30) + 4} GiB free, {free >> 30} GiB available")


def _rev(start, count, b, dev):
    """rev_b(i) for i in [start, start + count): independent torch shift loop."""
    idx = torch.arange(start, start + count, dtype=torch.int64, device=dev)
    r = torch.zeros_like(idx)
    for _ in range(b):
        r = (r << 1) | (idx & 1)
        idx >>= 1
    return r


def _words(t):
    """[n, w] integer view of an array of n elements (raw bits)."""
    E = t.element_size()
    if E == 4:
        return t.view(torch.int32).view(-1, 1)
    return t.view(torch.int64).view(-1, E // 8)


def _random_bits(n, dtype, dev):
    E = torch.empty(0, dtype=dtype).element_size()
    return torch.empty(n * E, dtype=torch.uint8, device=dev).random_(0, 256).view(dtype)


def _check_vs_device_oracle(x, out, b, base=0, total_bits=None):
    """out[j] == x[rev(j)] for every j, 2^CHUNK_BITS slots at a time.  With
    base/total_bits, `out` is the slice [base, base + len) of a 2^total_bits
    permutation whose full source is x."""
    tb = b if total_bits is None else total_bits
    xw, ow = _words(x), _words(out)
    n = ow.shape[0]
    step = 1 << CHUNK_BITS
    for s in range(0, n, step):
        c = min(step, n - s)
        r = _rev(base + s, c, tb, x.device)
        assert torch.equal(ow[s:s + c], xw.index_select(0, r)), f"mismatch in slots [{s}, {s + c})"


@pytest.mark.parametrize("dtype,b,rows", [(torch.float64, 26, 1), (torch.float64, 28, 1),
                                          (torch.complex128, 26, 1), (torch.complex128, 27, 1),
                                          (torch.complex64, 16, 2048), (torch.float64, 20, 128)],
                         ids=["f64-26", "f64-28", "c128-26", "c128-27", "c64-16x2048",
                              "f64-20x128"])
def test_spread_grid_launches_every_element(cuda, dtype, b, rows):
    """Launches large enough for the spread grids (about 5 tiles per CTA
    instead of a persistent grid: bitrev_capi.cu oop_grid), single arrays and
    batched rows, every element against the device oracle."""
    from paper_1708_01873_b200 import _lib

    x = _random_bits(rows << b, dtype, cuda)
    out = torch.empty_like(x)
    if rows == 1:
        br.cobra_out_of_place(x, out, br.CobraConfig(0), b)
    else:
        br.bitrev_batched(x.view(rows, 1 << b), b, out.view(rows, 1 << b))
    torch.cuda.synchronize()
    assert _lib.last_tile()[1] in (0, 3)  # the register tile families
    for r in range(rows):
        n = 1 << b
        _check_vs_device_oracle(x[r * n:(r + 1) * n], out[r * n:(r + 1) * n], b)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.complex128],
                         ids=["f32", "f64", "c128"])
def test_cfg3_out_of_place_every_element(cuda, dtype):
    b = 30
    E = torch.empty(0, dtype=dtype).element_size()
    _need(cuda, 2 * (E << b) + (2 << 30))
    x = _random_bits(1 << b, dtype, cuda)
    out = torch.empty_like(x)
    br.cobra_out_of_place(x, out, br.CobraConfig(6), b)
    torch.cuda.synchronize()
    _check_vs_device_oracle(x, out, b)
    # the in-place path (tile pairs / cluster pairs) on the same bytes
    br.cobra_in_place(x, br.CobraConfig(6), b)
    torch.cuda.synchronize()
    assert torch.equal(_words(x), _words(out))


def test_cfg3_complex128_sentinel_pairs(cuda):
    """Element i = (i, ~i) as two u64 words; out[j] must be (rev j, ~rev j)."""
    b = 30
    _need(cuda, 2 * (16 << b) + (2 << 30))
    x = torch.empty(1 << b, dtype=torch.complex128, device=cuda)
    w = x.view(torch.int64).view(-1, 2)
    step = 1 << CHUNK_BITS
    for s in range(0, 1 << b, step):
        i = torch.arange(s, s + step, dtype=torch.int64, device=cuda)
        w[s:s + step, 0] = i
        w[s:s + step, 1] = ~i
    out = torch.empty_like(x)
    br.cobra_out_of_place(x, out, br.CobraConfig(6), b)
    torch.cuda.synchronize()
    ow = out.view(torch.int64).view(-1, 2)
    for s in range(0, 1 << b, step):
        r = _rev(s, step, b, cuda)
        assert torch.equal(ow[s:s + step, 0], r), s
        assert torch.equal(ow[s:s + step, 1], ~r), s


def test_cfg2_float64_payload_vs_cpu_oracle(cuda):
    b = 26
    n = 1 << b
    rng = np.random.default_rng(2)
    host = rng.standard_normal(n)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan])
    pos = rng.integers(0, n, 4096)
    host[pos] = special[pos % len(special)]
    bits = host.view(np.uint64)
    nanpos = rng.integers(0, n, 1024)  # NaNs with distinct payload bits
    bits[nanpos] = np.uint64(0x7FF0000000000001) + rng.integers(0, 1 << 50, 1024).astype(np.uint64)
    expect = orc.oracle_permute(host, b)
    a = torch.from_numpy(host.copy()).to(cuda)
    br.cobra_in_place(a, br.CobraConfig(6), b)
    got = a.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), expect.view(np.uint64))
    # out of place on the same payload
    src = torch.from_numpy(host).to(cuda)
    out = torch.empty_like(src)
    br.cobra_out_of_place(src, out, br.CobraConfig(6), b)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), expect.view(np.uint64))


def test_cfg4_full_batch_vs_cpu_oracle(cuda):
    b, rows = 16, 4096
    rng = np.random.default_rng(4)
    host = rng.integers(0, 1 << 63, (rows, 1 << b), dtype=np.int64, endpoint=False) \
        .view(np.complex64).reshape(rows, -1)
    rev = orc.rev_index_array(b)
    expect = host[:, rev]
    x = torch.from_numpy(host).to(cuda)
    out = br.bitrev_batched(x, b)
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.int64), expect.view(np.int64))
    br.bitrev_batched_inplace(x, b)
    assert np.array_equal(x.cpu().numpy().view(np.int64), expect.view(np.int64))


def test_cfg5_plan_2p31_complex64_eight_ranks(cuda):
    """The sharded plan's kernels (pack with 4 exchange rounds, unpack) for 8
    emulated ranks on a 2^31-element complex64 array, every element."""
    b, G, chunks = 31, 8, 4
    _need(cuda, 3 * (8 << b))
    x = _random_bits(1 << b, torch.complex64, cuda)
    outs = sharded.emulate_sharded(x, b, G, chunks)
    S = 1 << (b - 3)
    for d, o in enumerate(outs):
        _check_vs_device_oracle(x, o, b - 3, base=d * S, total_bits=b)


@pytest.mark.parametrize("G,mode", [(2, "nccl"), (4, "nccl"), (8, "nccl"), (8, "p2p")])
def test_cfg5_full_size_2p32_complex64(cuda, G, mode):
    """Config 5 at its BASELINE size: 2^32 complex64 (32 GiB) over G emulated
    ranks, every element.  "nccl" = the pack kernel with 4 exchange rounds and
    the per-round unpack (sharded_bitrev's device steps; at G = 2 each shard
    holds 2^31 elements); "p2p" = the fused scatter into G receive buffers
    and the unpack (sharded_bitrev_p2p's device steps)."""
    b = 32
    _need(cuda, 3 * (8 << b) + (8 << b) // 4)
    x = _random_bits(1 << b, torch.complex64, cuda)
    g = G.bit_length() - 1
    if mode == "nccl":
        outs = sharded.emulate_sharded(x, b, G, 4)
    else:
        outs = sharded.emulate_sharded_p2p(x, b, G)
    S = 1 << (b - g)
    for d in range(G):
        _check_vs_device_oracle(x, outs[d], b - g, base=d * S, total_bits=b)
        outs[d] = None
        gc.collect()


@pytest.mark.parametrize("E", [4, 8, 16])
@pytest.mark.parametrize("g", [0, 1, 2, 3])
@pytest.mark.parametrize("bl", [3, 5, 12])
def test_unpack_vector_and_generic_forms(cuda, E, g, bl):
    """bitrev_sharded_unpack: the vector kernel (C*E >= 16) and the
    element-wise form (tiny chunks) both give dst[k*G + rev_g(r)] = recv[r*C + k]."""
    if g > bl:
        pytest.skip("g > b_local")
    dtype = {4: torch.int32, 8: torch.int64, 16: torch.complex128}[E]
    n = 1 << bl
    recv = _random_bits(n, dtype, cuda)
    out = torch.empty_like(recv)
    sharded._unpack(recv, bl, g, out)
    G, C = 1 << g, 1 << (bl - g)
    rw, ow = _words(recv), _words(out)
    for r in range(G):
        assert torch.equal(ow[orc.rev_naive(r, g)::G], rw[r * C:(r + 1) * C]), r


@pytest.mark.parametrize("E", [4, 8, 16])
@pytest.mark.parametrize("bl,g,kb", [(14, 1, 0), (14, 1, 3), (14, 1, 7), (13, 1, 4), (16, 2, 2),
                                      (17, 3, 1), (20, 3, 4)])
def test_pack_layout(cuda, E, bl, g, kb):
    """bitrev_sharded_pack: the local reversal laid out [c][d][k'] -- through
    the rectangular pack tiles, or the square scatter tiles when a sub-chunk
    is shorter than a rectangular destination row (kb = 7) or the shard is
    narrower than a rectangular tile (b_local = 13)."""
    dtype = {4: torch.int32, 8: torch.int64, 16: torch.complex128}[E]
    x = _random_bits(1 << bl, dtype, cuda)
    send = sharded._pack(x, bl, g, kb)
    G, K = 1 << g, 1 << kb
    L = _words(br.oracle_permute(x, bl))
    expect = L.view(G, K, -1, L.shape[1]).transpose(0, 1).reshape(-1, L.shape[1])
    assert torch.equal(_words(send), expect)
