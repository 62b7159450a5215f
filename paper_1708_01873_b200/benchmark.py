"""The reference's benchmark API on the device (src/bench.py:69-110, 131-132,
189-357, 370-433): BenchConfig, validate_config, SkipMethod, run_benchmark,
CobraTuneResult and tune_cobra, with the same fields, validation messages,
seeded per-replicate refills, skip rules and record schema, so a caller of
`bitrev.run_benchmark(BenchConfig(...))` or `bitrev.tune_cobra(...)` can switch
to this package unchanged and feed the records to the reference's CSV tools.

What differs is the clock: every sample is measured with CUDA events on the
current stream around the method's kernel launches (the refill, an H2D copy
of the reference's fill, and an optional L2 flush sit outside the events).
Small sizes loop the call an odd number of times so a sample spans at least
a millisecond, as the reference does (src/bench.py:312-320).
write_gbs_sidecar adds the bandwidth columns the reference schema lacks.
"""

from __future__ import annotations

import csv
import logging
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _core, _lib
from .bits import MAX_BITS
from .harness import (
    ELEMENT_KINDS,
    METHOD_IDS,
    NUMPY_KINDS,
    BenchmarkRecord,
    fill_numpy,
    make_method,
    make_record,
)
from .permutations import default_cobra_q
from .recursive import RecursionPolicy
from .schedule import swap_count
from .verify import oracle_permute

log = logging.getLogger("bitrev_b200.bench")

_MIN_SAMPLE_S = 1e-3   # a timed sample spans at least this long
_LOOP_CAP = 100001
_FLUSH_BYTES = 512 << 20


@dataclass
class BenchConfig:
    """One benchmark invocation (the reference's fields, src/bench.py:69-88),
    plus two device knobs: flush_l2 evicts the array from the L2 before every
    replicate, device picks the GPU (default: the current one)."""

    methods: tuple[str, ...] = METHOD_IDS
    b_min: int = 8
    b_max: int = 20
    replicates: int = 100
    warmup: int = 3
    element_kind: str = "pair"
    cobra_q: int | None = None
    tune_cobra_q: bool = False
    base_bits: int = 9
    depth_limit: int = 1
    threads: int = 0
    seed: int = 0
    verify: bool = False
    out: str | None = None
    unrolled_max_bits: int = 16
    memory_cap_bytes: int = 1 << 30
    flush_l2: bool = True
    device: str | None = None


def validate_config(cfg: BenchConfig) -> None:
    """Reject a bad configuration before anything runs (src/bench.py:91-110)."""
    if not cfg.methods:
        raise ValueError("no methods selected")
    unknown = [m for m in cfg.methods if m not in METHOD_IDS]
    if unknown:
        raise ValueError(f"unknown methods: {unknown}; choose from {METHOD_IDS}")
    if not (1 <= cfg.b_min <= cfg.b_max <= MAX_BITS):
        raise ValueError(f"need 1 <= b_min <= b_max <= {MAX_BITS}")
    if cfg.replicates < 1:
        raise ValueError("replicates must be >= 1")
    if cfg.warmup < 0:
        raise ValueError("warmup must be >= 0")
    if cfg.element_kind not in ELEMENT_KINDS:
        raise ValueError(f"unknown element kind {cfg.element_kind!r}")
    if cfg.cobra_q is not None and cfg.cobra_q < 0:
        raise ValueError("cobra_q must be >= 0")
    if cfg.memory_cap_bytes < 1:
        raise ValueError("memory_cap_bytes must be positive")
    RecursionPolicy(cfg.base_bits, cfg.depth_limit)


class SkipMethod(Exception):
    """A (method, size) cell that cannot or should not run (src/bench.py:131-132)."""


class _Cell:
    """One (method, b) cell: device array, optional destination, the launch."""

    def __init__(self, method: str, b: int, cfg: BenchConfig, dev: torch.device, q: int):
        kind = cfg.element_kind
        esize = NUMPY_KINDS[kind].itemsize
        n = 1 << b
        # the reference's footprint estimate and skip rules (src/bench.py:205-224)
        extra = n * esize if method in ("stockham", "cobra") else 0
        if method == "unrolled":
            if b > cfg.unrolled_max_bits:
                raise SkipMethod(f"unrolled is capped at b={cfg.unrolled_max_bits}")
            extra = 16 * swap_count(b)
        est = n * esize + extra
        if est > cfg.memory_cap_bytes:
            raise SkipMethod(f"estimated {est / 2**20:.0f} MiB exceeds the "
                             f"{cfg.memory_cap_bytes / 2**20:.0f} MiB cap")
        if method in ("cobra", "cobra_inplace") and 2 * q > b:
            raise SkipMethod(f"cobra q={q} needs 2q <= b")
        try:
            self.array = torch.empty(n, dtype=ELEMENT_KINDS[kind], device=dev)
            self.dest = torch.empty_like(self.array) if method == "cobra" else None
        except torch.cuda.OutOfMemoryError as e:
            raise SkipMethod(f"allocation failed: {e}") from e
        self.method, self.b = method, b
        if method == "cobra":
            from .permutations import CobraConfig, cobra_out_of_place

            ccfg = CobraConfig(q)
            self.run = lambda: cobra_out_of_place(self.array, self.dest, ccfg, b)
        elif method == "cobra_inplace":
            from .permutations import CobraConfig, cobra_in_place

            ccfg = CobraConfig(q)
            self.run = lambda: cobra_in_place(self.array, ccfg, b)
        else:
            fn = make_method(method, base_bits=cfg.base_bits, depth_limit=cfg.depth_limit,
                             threads=cfg.threads)
            self.run = lambda: fn(self.array, b)

    def result(self) -> torch.Tensor:
        return self.dest if self.dest is not None else self.array


def _refill(cell: _Cell, cfg: BenchConfig, replicate: int) -> None:
    host = fill_numpy(1 << cell.b, cfg.element_kind, cfg.seed, cell.method, cell.b, replicate)
    cell.array.copy_(torch.from_numpy(host))


def _time_launches(run, k: int, stream) -> float:
    """Seconds per call of k back-to-back calls, CUDA events on `stream`."""
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(k):
        run()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / 1e3 / k


def _loop_count(run, stream) -> int:
    """Odd call count so a sample spans >= 1 ms; in-place methods (involutions)
    then end in the permuted state, as in src/bench.py:312-320."""
    dt = _time_launches(run, 1, stream)
    k = min(_LOOP_CAP, max(1, math.ceil(_MIN_SAMPLE_S / max(dt, 1e-8))))
    return k if k % 2 else k + 1


def _resolve_q(method: str, b: int, cfg: BenchConfig) -> int:
    if cfg.cobra_q is not None:
        return cfg.cobra_q
    if cfg.tune_cobra_q and method in ("cobra", "cobra_inplace"):
        cands = list(range(0, min(b // 2, 8) + 1))
        res = tune_cobra(b, cands, replicates=3, element_kind=cfg.element_kind, seed=cfg.seed,
                         variant=method)
        log.info("%s b=%d: tuned q=%d", method, b, res.best_q)
        return res.best_q
    return default_cobra_q(b)


def run_benchmark(cfg: BenchConfig) -> list[BenchmarkRecord]:
    """Run the configured grid on the device; one record per replicate
    (src/bench.py:323-357).  Method order is shuffled per size with the
    reference's generator; unrunnable cells are skipped with a logged notice;
    with cfg.verify the final state of every cell is compared with the oracle
    on the last replicate's fill (RuntimeError on any difference)."""
    validate_config(cfg)
    dev = torch.device(cfg.device) if cfg.device is not None else _core.require_cuda()
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(_FLUSH_BYTES, dtype=torch.uint8, device=dev) if cfg.flush_l2 else None
    order = np.random.default_rng(cfg.seed)
    records: list[BenchmarkRecord] = []
    with torch.cuda.device(dev):
        for b in range(cfg.b_min, cfg.b_max + 1):
            methods = list(cfg.methods)
            order.shuffle(methods)
            for method in methods:
                try:
                    cell = _Cell(method, b, cfg, dev, _resolve_q(method, b, cfg))
                except SkipMethod as skip:
                    log.warning("skipping %s at b=%d: %s", method, b, skip)
                    continue
                _refill(cell, cfg, -1)
                for _ in range(cfg.warmup):
                    cell.run()
                k = _loop_count(cell.run, stream) if b < 12 else 1
                for rep in range(cfg.replicates):
                    _refill(cell, cfg, rep)
                    if flush is not None:
                        flush.zero_()
                    records.append(make_record(method, b, rep, _time_launches(cell.run, k, stream)))
                if cfg.verify:
                    expect = oracle_permute(
                        torch.from_numpy(fill_numpy(1 << b, cfg.element_kind, cfg.seed, method, b,
                                                    cfg.replicates - 1)).to(dev), b)
                    got = cell.result()
                    if not torch.equal(got.view(torch.uint8), expect.view(torch.uint8)):
                        raise RuntimeError(f"{method} at b={b} left a non-permuted array")
                    log.info("verified %s at b=%d against the oracle", method, b)
                del cell
    return records


@dataclass
class CobraTuneResult:
    """Per-candidate timing table and the winning block width
    (src/bench.py:369-377).  `effective` maps each candidate q to the
    (tile bits, staging path) the device actually ran for it."""

    b: int
    variant: str
    best_q: int
    means: dict[int, float]
    records: list[BenchmarkRecord] = field(default_factory=list)
    effective: dict[int, tuple[int, int]] = field(default_factory=dict)


def tune_cobra(b: int, q_candidates, replicates: int = 5, element_kind: str = "pair",
               seed: int = 0, variant: str = "cobra") -> CobraTuneResult:
    """Time each candidate block width and keep the fastest mean, ties toward
    the smaller q (src/bench.py:380-433).

    On the device the block width is the shared-memory tile bits Q of the
    variant's kernel family: a candidate the family instantiates for this
    element size runs with exactly that Q forced; any other candidate (the
    CPU-only widths 0..2, or past the family's range) runs the library's
    default selection, and `effective[q]` records what ran.  Rows are
    benchmark records with method id cobra_q<q> / cobra_inplace_q<q>."""
    q_candidates = list(q_candidates)
    if not q_candidates:
        raise ValueError("q_candidates must not be empty")
    bad = [q for q in q_candidates if q < 0 or 2 * q > b]
    if bad:
        raise ValueError(f"candidates {bad} violate 0 <= 2q <= b for b={b}")
    if variant not in ("cobra", "cobra_inplace"):
        raise ValueError(f"variant must be cobra or cobra_inplace, not {variant!r}")
    if replicates < 1:
        raise ValueError("replicates must be >= 1")
    if element_kind not in ELEMENT_KINDS:
        raise ValueError(f"unknown element kind {element_kind!r}")
    dev = _core.require_cuda()
    stream = torch.cuda.current_stream(dev)
    inplace = variant == "cobra_inplace"
    E = NUMPY_KINDS[element_kind].itemsize
    cfg = BenchConfig(methods=(variant,), element_kind=element_kind, seed=seed,
                      memory_cap_bytes=1 << 62)
    cell = _Cell(variant, b, cfg, dev, 0)
    old_q = _lib.get_tile_bits(E, inplace)
    restore = 0 if old_q == _lib_default(E, inplace) else old_q
    result = CobraTuneResult(b, variant, -1, {})
    try:
        for q in q_candidates:
            try:
                _lib.set_tile_bits(E, inplace, q)
            except _lib.BitrevError:
                _lib.set_tile_bits(E, inplace, 0)  # not instantiated: library default
            _refill(cell, cfg, -1)
            cell.run()
            torch.cuda.synchronize(dev)
            result.effective[q] = _lib.last_tile()
            k = _loop_count(cell.run, stream) if b < 12 else 1
            samples = []
            for rep in range(replicates):
                _refill(cell, cfg, rep)
                dt = _time_launches(cell.run, k, stream)
                samples.append(dt)
                result.records.append(make_record(f"{variant}_q{q}", b, rep, dt))
            result.means[q] = sum(samples) / len(samples)
    finally:
        _lib.set_tile_bits(E, inplace, restore)
    result.best_q = min(result.means, key=lambda q: (result.means[q], q))
    return result


def _lib_default(E: int, inplace: bool) -> int:
    cur = _lib.get_tile_bits(E, inplace)
    _lib.set_tile_bits(E, inplace, 0)
    d = _lib.get_tile_bits(E, inplace)
    _lib.set_tile_bits(E, inplace, cur)
    return d


GBS_HEADER = ("method", "b", "n", "replicate", "elem_bytes", "bytes_moved", "gb_per_s",
              "gelem_per_s")


def write_gbs_sidecar(records: list[BenchmarkRecord], path, element_kind: str = "pair") -> None:
    """Bandwidth columns for a record table: one row per
    record, effective GB/s = 2*n*elem_bytes / elapsed_s and Gelem/s; the
    reference CSV stays byte-for-byte its own schema (write_csv)."""
    E = NUMPY_KINDS[element_kind].itemsize
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(GBS_HEADER)
        for r in records:
            moved = 2 * r.n * E
            w.writerow([r.method, r.b, r.n, r.replicate, E, moved,
                        repr(moved / r.elapsed_s / 1e9), repr(r.n / r.elapsed_s / 1e9)])
