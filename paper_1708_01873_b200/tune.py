"""Tile autotuner: the GPU analogue of tune_cobra (src/bench.py:380-433).

The reference tunes COBRA's block width q per size by timing candidates and
keeping the fastest mean (ties toward the smaller buffer).  Here the knobs are
the shared-memory tile bits Q and the staging path (0 = register staging,
1 = per-row cp.async.bulk ring, 2 = TMA tensor-map ring, 3 = rectangular
register tiles, out of place only, 4 = element-granular cp.async pipeline, in
place only) of each kernel family;
the output never depends on them.  Candidates are timed in interleaved rounds
(every candidate once per round) with CUDA events, so clock or box drift during
the run hits all candidates alike.  Records use the reference CSV schema
(method id "gpu_q<Q>_p<path>").
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _core, _lib
from .harness import BenchmarkRecord, make_record

QS = {4: (5, 6, 7), 8: (4, 5, 6), 16: (3, 4, 5, 6)}
PATHS = (0, 1, 2)
# path 3: rectangular out-of-place tiles, q = destination-run bits QX
RECT_QS = {4: (6, 7, 8), 8: (5, 6, 7), 16: (4, 5, 6, 7)}
DTYPES = {4: torch.float32, 8: torch.float64, 16: torch.complex128}


@dataclass
class TileTuneResult:
    b: int
    elem_bytes: int
    inplace: bool
    best: tuple[int, int]
    gbs: dict[tuple[int, int], float]
    records: list[BenchmarkRecord] = field(default_factory=list)


def tune_tiles(elem_bytes: int, inplace: bool, b: int, candidates=None, rounds: int = 5,
               launches: int = 5, apply: bool = True, device=None,
               batch: int = 1) -> TileTuneResult:
    """Time every (q, path) candidate on `batch` random rows of 2^b elements;
    optionally make the fastest the library's setting for (elem_bytes, family)."""
    if elem_bytes not in QS:
        raise ValueError("tile kernels exist for 4, 8 and 16-byte elements")
    cands = list(candidates) if candidates is not None else [
        (q, p) for q in QS[elem_bytes] for p in PATHS if 2 * q <= b]
    if candidates is None and not inplace:
        cands += [(q, 3) for q in RECT_QS[elem_bytes] if q + 5 <= b]
    if not cands:
        raise ValueError(f"no candidate tile widths for b={b}")
    bad = [q for q, p in cands
           if (p == 3 and (inplace or q not in RECT_QS[elem_bytes]))
           or (p != 3 and (2 * q > b or q not in QS[elem_bytes]))]
    if bad:
        raise ValueError(f"candidates {bad} are not valid tile bits for b={b}")
    dev = torch.device(device) if device is not None else _core.require_cuda()
    n = 1 << b
    x = torch.empty(batch * n * elem_bytes, dtype=torch.uint8, device=dev).random_(0, 256)
    x = x.view(DTYPES[elem_bytes])
    if batch > 1:
        x = x.view(batch, n)
    y = None if inplace else torch.empty_like(x)
    old = (_lib.get_tile_bits(elem_bytes, inplace), _lib.get_tile_path(elem_bytes, inplace))
    samples: dict[tuple[int, int], list[float]] = {c: [] for c in cands}
    result = TileTuneResult(b, elem_bytes, inplace, cands[0], {})
    try:
        for rnd in range(rounds):
            for q, p in cands:
                _lib.set_tile_bits(elem_bytes, inplace, q)
                _lib.set_tile_path(elem_bytes, inplace, p)

                def run():
                    if inplace:
                        _core.launch_inplace(x, b)
                    else:
                        _core.launch_oop(x, y, b)

                run()
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(launches):
                    run()
                e.record()
                e.synchronize()
                dt = s.elapsed_time(e) / 1e3 / launches
                samples[(q, p)].append(dt)
                result.records.append(make_record(f"gpu_q{q}_p{p}", b, rnd, dt / batch))
    finally:
        _lib.set_tile_bits(elem_bytes, inplace, old[0])
        _lib.set_tile_path(elem_bytes, inplace, old[1])
    for c, ts in samples.items():
        ts = sorted(ts)
        result.gbs[c] = 2 * batch * n * elem_bytes / ts[len(ts) // 2] / 1e9
    result.best = max(cands, key=lambda c: (result.gbs[c], -c[0]))
    if apply:
        _lib.set_tile_bits(elem_bytes, inplace, result.best[0])
        _lib.set_tile_path(elem_bytes, inplace, result.best[1])
    return result
