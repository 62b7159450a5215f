"""CUDA-graph plans for repeated permutations on fixed buffers.

The reference methods are called again and again on the same arrays (the
benchmark protocol, an FFT pre-pass per frame).  On the GPU the per-call cost of
a small transform is host side: argument checks, tensor plumbing and the ctypes
launch.  A plan validates once, captures the launch (or a sequence of launches
over several batches) into a CUDA graph, and replays it with one
cudaGraphLaunch -- the B200 answer to a tracing compiler, with the kernels and
their order fixed at capture time.
"""

from __future__ import annotations

import torch

from . import _core, _lib
from .bits import check_width

_FFT_DTYPES = {torch.complex64: 8, torch.complex128: 16}


class BitrevPlan:
    """Captured bit reversal (optionally with fused DIT stages) on fixed tensors.

    src: CUDA tensor [2^b] or [batch, 2^b].  dst: None for in place, else a
    tensor of the same shape and dtype.  stages > 0 selects the FFT pre-pass
    (complex64/complex128, out of place).  The buffers must stay alive and
    keep their storage while the plan is used; refill them between replays.
    """

    def __init__(self, src: torch.Tensor, b: int, dst: torch.Tensor | None = None,
                 stages: int = 0, inverse: bool = False, replays_per_graph: int = 1):
        check_width(b)
        if not src.is_cuda or not src.is_contiguous():
            raise ValueError("plans need a contiguous CUDA tensor")
        if src.shape[-1] != (1 << b) or src.dim() not in (1, 2):
            raise ValueError(f"src length {src.shape[-1]} does not match 2**{b}")
        if dst is not None and (dst.shape != src.shape or dst.dtype != src.dtype
                                or not dst.is_contiguous() or dst.device != src.device):
            raise ValueError("dst must match src in shape, dtype, device and be contiguous")
        if dst is not None and _core.shares_memory(src, dst):
            raise ValueError("source and dest must not overlap")
        if stages and (dst is None or src.dtype not in _FFT_DTYPES):
            raise ValueError("fused FFT stages need an out-of-place complex64/complex128 plan")
        if replays_per_graph < 1:
            raise ValueError("replays_per_graph must be >= 1")
        self.src, self.dst, self.b = src, dst, b
        self.stages, self.inverse = stages, inverse
        self.batch = 1 if src.dim() == 1 else src.shape[0]
        self.elem = _core.elem_bytes(src)
        self.launches_per_replay = replays_per_graph
        dev = src.device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.device(dev), torch.cuda.stream(side):
            # warm: kernel attributes, occupancy caches, TMA encode paths.  An
            # in-place plan warms with two launches: the permutation is an
            # involution, so the caller's data comes back unchanged.
            self._launch()
            if dst is None:
                self._launch()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.device(dev), torch.cuda.graph(self.graph):
            for _ in range(replays_per_graph):
                self._launch()

    def _launch(self) -> None:
        n = 1 << self.b
        stream = _core._stream_ptr(self.src.device)
        if self.stages:
            _lib.call("bitrev_dit_prepass", self.src.data_ptr(), self.dst.data_ptr(), self.b,
                      self.elem, self.batch, n, n, self.stages, int(self.inverse), stream)
        elif self.dst is None:
            _lib.call("bitrev_inplace", self.src.data_ptr(), self.b, self.elem, self.batch, n,
                      stream)
        else:
            _lib.call("bitrev_oop", self.src.data_ptr(), self.dst.data_ptr(), self.b, self.elem,
                      self.batch, n, n, stream)

    def replay(self) -> torch.Tensor:
        """Run the captured launches on the current stream; returns the result
        tensor (dst, or src for in-place plans)."""
        self.graph.replay()
        return self.src if self.dst is None else self.dst


def make_plan(src: torch.Tensor, b: int, dst: torch.Tensor | None = None, **kw) -> BitrevPlan:
    """Build a BitrevPlan (see its docstring)."""
    return BitrevPlan(src, b, dst, **kw)
