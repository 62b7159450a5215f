"""Method registry, element kinds, input fills and the benchmark record schema
(the hot-path parts of src/bench.py).

make_method (src/bench.py:135-185) is the uniform (array, b) adapter the
reference's tests and acceptance suite drive; METHOD_IDS / ELEMENT_KINDS /
fill keep the reference's ids, dtypes and seeded distributions so GPU and CPU
runs see identical inputs.  Records use the reference CSV schema
(src/bench.py:436-473), so the reference tooling (read_csv, plotkit) reads GPU
series unchanged; the benchmark driver itself is benchmark.py.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from .parallel import ParallelConfig, parallel_semi_recursive_permute
from .permutations import (
    CobraConfig,
    bytetable_permute,
    cobra_in_place,
    cobra_out_of_place,
    default_cobra_q,
    naive_bitwise_permute,
    pair_bitwise_permute,
    stockham_permute,
    xor_permute,
)
from .recursive import RecursionPolicy, recursive_permute, semi_recursive_permute
from .schedule import apply_schedule, cached_schedule

METHOD_IDS = (
    "stockham",
    "bitwise",
    "bytewise",
    "pair",
    "cobra",
    "cobra_inplace",
    "xor",
    "unrolled",
    "recursive",
    "semirecursive",
    "parallel",
)

ELEMENT_KINDS = {
    "pair": torch.complex128,  # 16-byte two-component float cell (the default)
    "f8": torch.float64,
    "f4": torch.float32,
    "i8": torch.int64,
}

NUMPY_KINDS = {
    "pair": np.dtype(np.complex128),
    "f8": np.dtype(np.float64),
    "f4": np.dtype(np.float32),
    "i8": np.dtype(np.int64),
}


def make_method(method: str, *, cobra_q: int | None = None, base_bits: int = 9,
                depth_limit: int = 1, threads: int = 0) -> Callable:
    """Uniform (array, b) adapter over every method id (src/bench.py:135-185).

    In-place methods mutate and return None; "cobra" returns a new array.
    """
    if method == "stockham":
        return lambda a, b: stockham_permute(a, b)
    if method == "bitwise":
        return lambda a, b: naive_bitwise_permute(a, b)
    if method == "bytewise":
        return lambda a, b: bytetable_permute(a, b)
    if method == "pair":
        return lambda a, b: pair_bitwise_permute(a, b)
    if method == "xor":
        return lambda a, b: xor_permute(a, b)
    if method == "unrolled":
        return lambda a, b: apply_schedule(a, cached_schedule(b))
    if method == "cobra":

        def run_cobra(a, b):
            dest = torch.empty_like(a) if isinstance(a, torch.Tensor) else np.empty_like(a)
            q = default_cobra_q(b) if cobra_q is None else cobra_q
            cobra_out_of_place(a, dest, CobraConfig(q), b)
            return dest

        return run_cobra
    if method == "cobra_inplace":

        def run_cobra_ip(a, b):
            q = default_cobra_q(b) if cobra_q is None else cobra_q
            cobra_in_place(a, CobraConfig(q), b)

        return run_cobra_ip
    if method == "recursive":
        return lambda a, b: recursive_permute(a, b, RecursionPolicy(base_bits, None))
    if method == "semirecursive":
        return lambda a, b: semi_recursive_permute(a, b, base_bits, depth_limit)
    if method == "parallel":
        pcfg = ParallelConfig(threads=threads, base_bits=base_bits)
        return lambda a, b: parallel_semi_recursive_permute(a, b, pcfg)
    raise ValueError(f"unknown method {method!r}")


def fill_numpy(n: int, kind: str, seed: int, method: str, b: int, replicate: int) -> np.ndarray:
    """The reference's seeded fill (src/bench.py:299-309) as a new numpy array."""
    dtype = NUMPY_KINDS[kind]
    ss = np.random.SeedSequence([seed, METHOD_IDS.index(method), b, replicate + 1])
    rng = np.random.default_rng(ss)
    out = np.empty(n, dtype=dtype)
    if dtype.kind == "c":
        out.real = rng.standard_normal(n)
        out.imag = rng.standard_normal(n)
    elif dtype.kind == "f":
        out[:] = rng.standard_normal(n, dtype=dtype)
    else:
        out[:] = rng.integers(0, 1 << 62, n, dtype=dtype)
    return out


# ---------------------------------------------------------------------------
# records and CSV (src/bench.py:112-128, 436-473)


@dataclass
class BenchmarkRecord:
    method: str
    b: int
    replicate: int
    elapsed_s: float
    per_element_s: float

    @property
    def n(self) -> int:
        return 1 << self.b


def make_record(method: str, b: int, replicate: int, elapsed_s: float) -> BenchmarkRecord:
    return BenchmarkRecord(method, b, replicate, elapsed_s, elapsed_s / (1 << b))


CSV_HEADER = ("method", "b", "n", "replicate", "elapsed_s", "per_element_s")


def write_csv(records: list[BenchmarkRecord], path) -> None:
    """Reference schema; floats via repr for an exact round trip."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for r in records:
            w.writerow([r.method, r.b, r.n, r.replicate, repr(r.elapsed_s), repr(r.per_element_s)])


def read_csv(path) -> list[BenchmarkRecord]:
    records = []
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = tuple(next(reader, ()))
        if header != CSV_HEADER:
            raise ValueError(f"{path}: unexpected header {header!r}")
        for lineno, row in enumerate(reader, start=2):
            if len(row) != len(CSV_HEADER):
                raise ValueError(f"{path}:{lineno}: expected {len(CSV_HEADER)} fields")
            method, b, n, rep, el, pe = row
            rec = BenchmarkRecord(method, int(b), int(rep), float(el), float(pe))
            if rec.n != int(n):
                raise ValueError(f"{path}:{lineno}: n={n} does not match 2**{b}")
            records.append(rec)
    return records
