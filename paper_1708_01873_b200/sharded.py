"""One 2^b array sharded by its top g index bits over G = 2^g ranks.

No reference counterpart (the reference is single-host); this
is BASELINE config 5.  Rank r owns global indices r*2^(b-g) + j.  Writing
j = m*G + l (l = low g bits), rev_b(r*2^(b-g) + j) = rev_{b-g}(j)*G + rev_g(r)
and rev_{b-g}(j) = rev_g(l)*2^(b-2g) + rev_{b-2g}(m), so:

  1. local:  L = bitrev_{b-g}(shard)            -- the single-GPU tile kernel;
             L is already G contiguous chunks of C = 2^(b-2g) elements,
             chunk d destined for rank d = rev_g(l);
  2. exchange: all_to_all_single, equal splits  -- NCCL over NVLink/NVSwitch;
             rank d receives recv[r] = L_r[d];
  3. local:  out[k*G + rev_g(r)] = recv[r][k]    -- bitrev_sharded_unpack.

sharded_bitrev_p2p fuses steps 1 and 2 for ranks that share peer-mapped
memory (one NVLink/NVSwitch node): the tile kernel's destination rows are
stored straight into the owning rank's receive buffer.

Requires b >= 2g.  Each element crosses HBM twice per local step and NVLink
once (unless it stays on its own rank: 1/G of the data).
"""

from __future__ import annotations

import ctypes
from typing import Callable

import torch
import torch.distributed as dist

from . import _core, _lib
from .bits import check_width


def shard_bits(world_size: int) -> int:
    g = world_size.bit_length() - 1
    if world_size < 1 or (1 << g) != world_size:
        raise ValueError(f"world size must be a power of two, got {world_size}")
    return g


def check_plan(b: int, world_size: int) -> int:
    check_width(b)
    g = shard_bits(world_size)
    if 2 * g > b:
        raise ValueError(f"sharded bit reversal needs b >= 2*log2(G): b={b}, G={world_size}")
    return g


def _local_bitrev(shard: torch.Tensor, b_local: int) -> torch.Tensor:
    out = torch.empty_like(shard)
    _core.launch_oop(shard, out, b_local)
    return out


def _pack(shard: torch.Tensor, b_local: int, g: int, kb: int) -> torch.Tensor:
    """Step 1 into a new send buffer laid out [sub-chunk c][destination d][k']
    (bitrev_sharded_pack); kb = 0 is the plain local reversal."""
    send = torch.empty_like(shard)
    with torch.cuda.device(shard.device):
        _lib.call("bitrev_sharded_pack", shard.data_ptr(), send.data_ptr(), b_local, g, kb,
                  _core.elem_bytes(shard), _core._stream_ptr(shard.device))
    return send


def _unpack(recv: torch.Tensor, b_local: int, g: int, out: torch.Tensor) -> None:
    """Step 3 into `out` (contiguous, recv-sized): out[k*G + rev_g(r)] = recv[r*C + k]."""
    with torch.cuda.device(recv.device):
        _lib.call("bitrev_sharded_unpack", recv.data_ptr(), out.data_ptr(), b_local, g,
                  _core.elem_bytes(recv), _core._stream_ptr(recv.device))


def _all_to_all_single(out: torch.Tensor, inp: torch.Tensor, group):
    """Equal-split all-to-all of one round (async); returns the work handle."""
    return dist.all_to_all_single(out, inp, group=group, async_op=True)


def sharded_bitrev(local: torch.Tensor, b: int, group=None, *, chunks: int = 1,
                   pack: Callable | None = None,
                   unpack: Callable | None = None,
                   phases: dict | None = None) -> torch.Tensor:
    """Bit-reverse the global 2^b array whose rank-r shard is `local`.

    Returns this rank's shard of the permuted array (a new tensor).

    Step 1 (pack) writes the local reversal as `chunks` = K rows of G*S
    elements (S = C/K): row c holds sub-chunk c of every destination chunk, so
    each row is the equal-split input of one `all_to_all_single` round.  The K
    rounds are issued asynchronously; round c is interleaved (step 3) into the
    contiguous output slice [c*S*G, (c+1)*S*G) as soon as it lands, while the
    later rounds are still on the wire.  With K = 1 the pack is the plain
    local reversal (bitrev_oop).

    `pack(shard, b_local, g, kb)` and `unpack(recv, bits, g, out)` default to
    the CUDA kernels; they are injectable so that the exchange itself (the
    product's all_to_all_single rounds) runs under gloo on CPU tensors.
    `phases`, if given, receives CUDA events "t0", "packed", "exchanged",
    "done" recorded on the current stream (K = 1 only, for phase timing).
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    g = check_plan(b, world)
    b_local = b - g
    if local.dim() != 1 or local.shape[0] != (1 << b_local):
        raise ValueError(f"local shard length {local.shape[0]} does not match 2**{b_local}")
    C = 1 << (b_local - g)
    if chunks < 1 or chunks & (chunks - 1) or chunks > C:
        raise ValueError(f"chunks must be a power of two in 1..{C}, got {chunks}")
    if chunks > 1 and (C // chunks < 64 or b_local < 12):
        # rounds are a pipelining knob only (the output does not depend on
        # them); sub-chunks shorter than a tile row cannot be packed, and
        # shards this small gain nothing from overlap
        chunks = 1
    kb = chunks.bit_length() - 1
    if (pack is None or unpack is None) and not local.is_cuda:
        raise ValueError("sharded_bitrev runs its local steps on the GPU: the shard must be a "
                         "CUDA tensor")
    pack = pack or _pack
    unpack = unpack or _unpack
    timed = phases is not None and local.is_cuda

    def mark(name):
        if timed:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream(local.device))
            phases[name] = ev

    mark("t0")
    send = pack(local.contiguous(), b_local, g, kb)
    mark("packed")
    if world == 1:
        mark("exchanged")
        mark("done")
        return send
    G = world
    sub = C // chunks
    recv = torch.empty_like(send)
    sv, rv = send.view(chunks, G * sub), recv.view(chunks, G * sub)
    works = [_all_to_all_single(rv[c], sv[c], group) for c in range(chunks)]
    out = torch.empty_like(send)
    for c in range(chunks):
        if works[c] is not None:
            works[c].wait()
        if c == 0 and chunks == 1:
            mark("exchanged")
        unpack(rv[c], b_local - kb, g, out[c * sub * G:(c + 1) * sub * G])
    if chunks > 1:
        mark("exchanged")
    mark("done")
    return out


def _scatter(local: torch.Tensor, b_local: int, g: int, rank: int, peers: list) -> None:
    """Steps 1+2 fused: local bitrev stored straight into the G receive buffers."""
    ptrs = (ctypes.c_void_p * len(peers))(*[p.data_ptr() for p in peers])
    with torch.cuda.device(local.device):
        _lib.call("bitrev_sharded_scatter", local.data_ptr(), ctypes.cast(ptrs, ctypes.c_void_p),
                  b_local, g, rank, _core.elem_bytes(local), _core._stream_ptr(local.device))


def sharded_bitrev_p2p(local: torch.Tensor, b: int, peer_recv: list, rank: int,
                       barrier: Callable) -> torch.Tensor:
    """Peer-memory variant of sharded_bitrev for one NVLink/NVSwitch node.

    peer_recv[d] is rank d's receive buffer (2^(b-g) elements) mapped into
    this process -- e.g. the peer views of a torch symmetric-memory allocation
    or CUDA IPC handles.  The local reversal writes its rows straight into the
    peers' buffers (bitrev_sharded_scatter: no send buffer, no NCCL pass);
    `barrier()` must order every rank's stores before any rank reads its
    buffer (a device-side or stream-synchronised cross-rank barrier); then the
    interleave runs locally, and a second barrier keeps every rank's next
    scatter out of the buffers until all unpacks have read them, so the same
    buffers can be reused call after call.  Returns this rank's shard of the
    permuted array.
    """
    world = len(peer_recv)
    g = check_plan(b, world)
    b_local = b - g
    if local.dim() != 1 or local.shape[0] != (1 << b_local):
        raise ValueError(f"local shard length {local.shape[0]} does not match 2**{b_local}")
    _scatter(local.contiguous(), b_local, g, rank, peer_recv)
    barrier()  # every rank's stores into my buffer are done
    out = torch.empty_like(local)
    _unpack(peer_recv[rank], b_local, g, out)
    # no rank may scatter its next call into my buffer before my unpack has
    # read it (write-after-read across calls on the same symmetric buffers)
    barrier()
    return out


def symmetric_recv(n: int, dtype, device, group=None):
    """Receive buffers for sharded_bitrev_p2p from torch symmetric memory.

    Returns (peer_views, barrier, handle): peer_views[d] is rank d's
    n-element buffer mapped into this process, barrier() is the handle's
    stream-ordered cross-rank barrier (it publishes the peers' stores), and
    the handle must be kept alive while the buffers are used.  Needs a node
    whose GPUs can map each other's memory (NVLink/NVSwitch); not exercised
    in the single-GPU test runs of this repo.
    """
    import torch.distributed._symmetric_memory as symm

    buf = symm.empty(n, dtype=dtype, device=device)
    hdl = symm.rendezvous(buf, group or dist.group.WORLD)
    peers = [hdl.get_buffer(r, (n,), dtype) for r in range(hdl.world_size)]
    return peers, (lambda: hdl.barrier()), (hdl, buf)


def emulate_sharded_p2p(global_array: torch.Tensor, b: int, world_size: int) -> list[torch.Tensor]:
    """All ranks of sharded_bitrev_p2p on ONE device: the peer table holds G
    local receive buffers, so the fused scatter kernel and the unpack run
    exactly as on a node (the stores just do not cross NVLink)."""
    g = check_plan(b, world_size)
    S = 1 << (b - g)
    recv = [torch.empty(S, dtype=global_array.dtype, device=global_array.device)
            for _ in range(world_size)]
    for r in range(world_size):
        _scatter(global_array[r * S:(r + 1) * S].contiguous(), b - g, g, r, recv)
    outs = []
    for d in range(world_size):
        out = torch.empty_like(recv[d])
        _unpack(recv[d], b - g, g, out)
        outs.append(out)
    return outs


def emulate_sharded(global_array: torch.Tensor, b: int, world_size: int,
                    chunks: int = 1) -> list[torch.Tensor]:
    """Run the three steps for `world_size` virtual ranks on ONE device, with
    the exchange done by device copies (rounds exactly like sharded_bitrev:
    the pack kernel's [c][d][k'] send layout, per-round unpack).  Used to
    check the plan's kernels on a single GPU; the real exchange is
    sharded_bitrev under torchrun."""
    g = check_plan(b, world_size)
    b_local = b - g
    S = 1 << b_local
    C = 1 << (b_local - g)
    G = world_size
    sub = C // chunks
    kb = chunks.bit_length() - 1
    sends = [_pack(global_array[r * S:(r + 1) * S].contiguous(), b_local, g, kb).view(chunks, G, sub)
             for r in range(G)]
    outs = []
    for d in range(G):
        out = torch.empty_like(global_array[:S])
        for c in range(chunks):
            recv = torch.cat([sends[r][c, d] for r in range(G)])
            _unpack(recv, b_local - kb, g, out[c * sub * G:(c + 1) * sub * G])
        outs.append(out)
    return outs
