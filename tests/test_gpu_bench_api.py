"""GPU tests of the reference-facing benchmark and schedule APIs.

* generate_swap_schedule / cached_schedule: the device generator
  (bitrev_swap_schedule) reproduces the reference's pair arrays in emission
  order (tests/golden/schedule_golden.json, produced by the reference's own
  generate_swap_schedule; /root/reference/pkg/tests/test_schedule.py:67-73);
* apply_schedule: an explicit schedule, a list with repeated indices (applied
  in list order like _apply_pairs) and out-of-range indices;
* run_benchmark(BenchConfig) over every method id with verify=True, the CSV
  round trip (and, when the reference package is installed in baseline/_ref,
  the reference's own read_csv), the GB/s sidecar;
* tune_cobra and tune_tiles.
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

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((Path(__file__).parent / "golden" / "schedule_golden.json").read_text())


@pytest.mark.parametrize("b", range(1, 23))
def test_generated_schedule_matches_reference_order(cuda, b):
    s = br.generate_swap_schedule(b)
    p = s.pairs
    assert p.is_cuda and p.dtype == torch.int64 and tuple(p.shape) == (GOLD["count"][str(b)], 2)
    raw = np.ascontiguousarray(p.cpu().numpy(), dtype="<i8").tobytes()
    assert hashlib.sha256(raw).hexdigest() == GOLD["sha256"][str(b)]
    if str(b) in GOLD["lists"]:
        assert p.tolist() == GOLD["lists"][str(b)]
    assert torch.equal(br.cached_schedule(b).pairs, p)


def test_golden_emission_order_small(cuda):
    assert br.generate_swap_schedule(2).pairs.tolist() == [[1, 2]]
    assert br.generate_swap_schedule(3).pairs.tolist() == [[1, 4], [3, 6]]
    assert br.generate_swap_schedule(4).pairs.tolist() == [
        [2, 4], [1, 8], [3, 12], [5, 10], [7, 14], [11, 13]]


def test_apply_explicit_schedules(cuda):
    b = 12
    x = torch.randint(0, 1 << 40, (1 << b,), device=cuda, dtype=torch.int64)
    # the generated pairs, replayed as an explicit (incomplete-flagged) list
    explicit = br.SwapSchedule(b, br.generate_swap_schedule(b).pairs.cpu().numpy())
    a = x.clone()
    br.apply_schedule(a, explicit)
    assert torch.equal(a, br.oracle_permute(x, b))
    # pairs sharing indices: the reference swaps them one after another
    pairs = np.array([[0, 5], [5, 9], [9, 0], [3, 3], [7, 1], [1, 7], [2, 4]], dtype=np.int64)
    host = x.cpu().numpy().copy()
    for i, j in pairs:
        host[i], host[j] = host[j], host[i]
    a = x.clone()
    br.apply_schedule(a, br.SwapSchedule(b, pairs))
    assert np.array_equal(a.cpu().numpy(), host)
    with pytest.raises(ValueError, match="index"):
        br.apply_schedule(x.clone(), br.SwapSchedule(b, np.array([[0, 1 << b]])))
    with pytest.raises(ValueError, match="index"):
        br.apply_schedule(x.clone(), br.SwapSchedule(b, np.array([[-1, 3]])))


def test_run_benchmark_every_method_verified(cuda, tmp_path):
    cfg = br.BenchConfig(b_min=3, b_max=13, replicates=2, warmup=1, verify=True)
    recs = br.run_benchmark(cfg)
    cells = {(r.method, r.b) for r in recs}
    assert cells == {(m, b) for m in br.METHOD_IDS for b in range(3, 14)}
    assert len(recs) == 2 * len(cells)
    assert all(r.elapsed_s > 0 and r.per_element_s == r.elapsed_s / r.n for r in recs)
    p = tmp_path / "gpu.csv"
    br.write_csv(recs, p)
    assert br.read_csv(p) == recs
    ref = ROOT / "baseline" / "_ref"
    if (ref / "bitrev" / "bench.py").exists():
        sys.path.insert(0, str(ref))
        try:
            import importlib

            ref_bench = importlib.import_module("bitrev.bench")
            back = ref_bench.read_csv(p)
            assert [(r.method, r.b, r.replicate, r.elapsed_s) for r in back] == \
                [(r.method, r.b, r.replicate, r.elapsed_s) for r in recs]
        except ImportError:
            pass
        finally:
            sys.path.remove(str(ref))
    side = tmp_path / "gpu_gbs.csv"
    br.write_gbs_sidecar(recs, side, cfg.element_kind)
    assert len(side.read_text().splitlines()) == len(recs) + 1


def test_run_benchmark_skip_rules(cuda):
    cfg = br.BenchConfig(methods=("unrolled", "cobra", "cobra_inplace"), b_min=17, b_max=17,
                         replicates=1, warmup=0, memory_cap_bytes=3 << 20, cobra_q=6)
    recs = br.run_benchmark(cfg)
    # unrolled is capped at 16 bits; cobra needs source + dest (4 MiB > 3 MiB);
    # cobra_inplace fits (2 MiB)
    assert {r.method for r in recs} == {"cobra_inplace"}
    # 2q <= b: q = 5 skips b = 8 and 9, runs b = 10
    cfg = br.BenchConfig(methods=("cobra",), b_min=8, b_max=10, replicates=1, warmup=0, cobra_q=5)
    assert {r.b for r in br.run_benchmark(cfg)} == {10}


@pytest.mark.parametrize("variant", ["cobra", "cobra_inplace"])
def test_tune_cobra(cuda, variant):
    res = br.tune_cobra(20, [0, 3, 4, 5, 6], replicates=2, variant=variant)
    assert isinstance(res, br.CobraTuneResult)
    assert res.b == 20 and res.variant == variant
    assert set(res.means) == {0, 3, 4, 5, 6} and res.best_q in res.means
    assert res.best_q == min(res.means, key=lambda q: (res.means[q], q))
    assert {r.method for r in res.records} == {f"{variant}_q{q}" for q in (0, 3, 4, 5, 6)}
    assert len(res.records) == 10 and set(res.effective) == set(res.means)
    # the library setting is restored afterwards
    x = torch.randint(0, 1 << 30, (1 << 20,), device=cuda, dtype=torch.int64)
    a = x.clone()
    br.cobra_in_place(a, br.CobraConfig(6), 20)
    assert torch.equal(a, br.oracle_permute(x, 20))


def test_run_benchmark_tuned_q(cuda):
    cfg = br.BenchConfig(methods=("cobra",), b_min=14, b_max=14, replicates=1, warmup=0,
                         tune_cobra_q=True, verify=True)
    assert len(br.run_benchmark(cfg)) == 1


@pytest.mark.parametrize("E,inplace", [(8, False), (16, True), (4, False)])
def test_tune_tiles(cuda, E, inplace):
    before = (br.get_tile_bits(E, inplace), br.get_tile_path(E, inplace))
    res = br.tune_tiles(E, inplace, 22, rounds=2, launches=2, apply=False)
    assert res.best in res.gbs and all(v > 0 for v in res.gbs.values())
    assert len(res.records) == 2 * len(res.gbs)
    assert (br.get_tile_bits(E, inplace), br.get_tile_path(E, inplace)) == before
    # every candidate gives the same bytes (output never depends on the tile)
    dtype = {4: torch.int32, 8: torch.int64, 16: torch.complex128}[E]
    x = torch.empty((1 << 22) * E, dtype=torch.uint8, device=cuda).random_(0, 256).view(dtype)
    want = br.oracle_permute(x, 22).view(torch.uint8)
    for q, p in list(res.gbs)[:4]:
        br.set_tile_bits(E, inplace, q)
        br.set_tile_path(E, inplace, p)
        try:
            if inplace:
                a = x.clone()
                br.cobra_in_place(a, br.CobraConfig(6), 22)
            else:
                a = torch.empty_like(x)
                br.cobra_out_of_place(x, a, br.CobraConfig(6), 22)
            assert torch.equal(a.view(torch.uint8), want), (q, p)
        finally:
            br.set_tile_bits(E, inplace, before[0])
            br.set_tile_path(E, inplace, before[1])


@pytest.mark.parametrize("b", [1, 5, 10])
def test_schedule_file_round_trip(cuda, tmp_path, b):
    s = br.generate_swap_schedule(b)
    path = tmp_path / f"sched{b}.bin"
    br.save_schedule(s, path)
    back = br.load_schedule(path)
    assert back.b == b and np.array_equal(back.pairs, s.pairs.cpu().numpy())
    raw = np.frombuffer(path.read_bytes()[9:], dtype="<u8").reshape(-1, 2)
    assert hashlib.sha256(raw.astype("<i8").tobytes()).hexdigest() == GOLD["sha256"][str(b)]
    x = torch.randint(0, 1 << 30, (1 << b,), device=cuda, dtype=torch.int64)
    a = x.clone()
    br.apply_schedule(a, back)
    assert torch.equal(a, br.oracle_permute(x, b))


def test_audit_swap_counts(cuda):
    assert br.audit_swap_counts(14) == {b: True for b in range(1, 15)}
    with pytest.raises(ValueError):
        br.audit_swap_counts(27)
