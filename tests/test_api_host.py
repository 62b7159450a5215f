"""Host-side behaviour of the reference-shaped API (no GPU needed): argument
validation with the reference's messages (tests/test_permutations.py:104-154,
tests/test_recursive.py:72-117 in the reference), the work-plan helpers of
src/parallel.py, recursion-plan traces, schedules, and the loud failure when no
CUDA device is present (there is no CPU path)."""

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from paper_1708_01873_b200 import recursive as rec


# --- validation -----------------------------------------------------------


@pytest.mark.parametrize("b", [0, 49, -1])
def test_width_domain(b):
    with pytest.raises(ValueError, match="bit width"):
        br.naive_bitwise_permute(np.zeros(4), b)
    with pytest.raises(ValueError, match="bit width"):
        br.check_width(b)


def test_length_and_ndim_messages():
    with pytest.raises(ValueError, match="does not match 2\\*\\*3"):
        br.xor_permute(np.zeros(9), 3)
    with pytest.raises(ValueError, match="must be 1-D"):
        br.cobra_in_place(np.zeros((2, 4)), br.CobraConfig(1), 3)
    with pytest.raises(ValueError, match="source length"):
        br.cobra_out_of_place(np.zeros(7), np.zeros(8), br.CobraConfig(1), 3)
    with pytest.raises(ValueError, match="dest length"):
        br.cobra_out_of_place(np.zeros(8), np.zeros(7), br.CobraConfig(1), 3)
    with pytest.raises(ValueError, match="does not match 2\\*\\*4"):
        br.recursive_permute(np.zeros(8), 4)


def test_cobra_config_checks():
    with pytest.raises(ValueError, match="q must be >= 0"):
        br.CobraConfig(-1)
    with pytest.raises(ValueError, match="2q <= b"):
        br.cobra_in_place(np.zeros(8), br.CobraConfig(2), 3)
    assert br.default_cobra_q(20) == 6 and br.default_cobra_q(5) == 2
    assert br.CobraConfig(3).buffer_size == 64


def test_overlap_rejected():
    a = np.zeros(16)
    with pytest.raises(ValueError, match="overlap"):
        br.cobra_out_of_place(a, a, br.CobraConfig(1), 4)
    t = torch.zeros(32)
    with pytest.raises(ValueError, match="overlap"):
        br.cobra_out_of_place(t[:16], t[8:24], br.CobraConfig(1), 4)


def test_scratch_rules():
    with pytest.raises(ValueError, match="scratch"):
        br.stockham_permute(np.zeros(16), 4, scratch=np.zeros(8))
    with pytest.raises(ValueError, match="scratch"):
        br.stockham_permute(np.zeros(16), 4, scratch=np.zeros(16, dtype=np.float32))
    with pytest.raises(ValueError, match="scratch"):
        br.recursive_permute(np.zeros(1 << 11), 11, br.RecursionPolicy(4), scratch=np.zeros(100))
    with pytest.raises(ValueError, match="dtype"):
        br.recursive_permute(np.zeros(1 << 11), 11, br.RecursionPolicy(4),
                             scratch=np.zeros(1 << 10, dtype=np.int32))
    with pytest.raises(ValueError, match="scratch"):
        br.even_odd_permute(np.zeros(16), 4, scratch=np.zeros(3))
    with pytest.raises(ValueError, match="scratch"):
        br.parallel_semi_recursive_permute(np.zeros(1 << 11), 11, scratch=np.zeros(10))


def test_policy_and_parallel_config_validation():
    with pytest.raises(ValueError):
        br.RecursionPolicy(0)
    with pytest.raises(ValueError):
        br.RecursionPolicy(4, depth_limit=0)
    with pytest.raises(ValueError):
        br.ParallelConfig(threads=-1)
    with pytest.raises(ValueError):
        br.ParallelConfig(depth_limit=2)


def test_transpose_validation():
    with pytest.raises(ValueError, match="h must be"):
        br.transpose_square_inplace(np.zeros(4), -1)
    with pytest.raises(ValueError, match="4\\*\\*2"):
        br.transpose_square_inplace(np.zeros(15), 2)
    br.transpose_square_inplace(np.zeros(1), 0)  # h = 0 is a no-op


def test_unknown_method():
    with pytest.raises(ValueError, match="unknown method"):
        br.make_method("nope")
    assert len(br.METHOD_IDS) == 11


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="CUDA"):
        br.cobra_in_place(np.arange(16.0), br.CobraConfig(1), 4)
    with pytest.raises(RuntimeError, match="CUDA"):
        br.cobra_out_of_place(torch.arange(16.0), torch.empty(16), br.CobraConfig(1), 4)


# --- work-plan helpers (reference tests/test_parallel.py) ------------------


@pytest.mark.parametrize("count,workers", [(1, 1), (7, 3), (64, 8), (100, 7), (5, 9)])
def test_chunk_ranges_partition(count, workers):
    chunks = br.chunk_ranges(count, workers)
    covered = [i for lo, hi in chunks for i in range(lo, hi)]
    assert covered == list(range(count))
    assert len(chunks) <= workers


@pytest.mark.parametrize("h", [2, 3, 4, 6, 9])
def test_transpose_tiles_own_each_cell_once(h):
    side = 1 << h
    owner = np.zeros((side, side), dtype=int)
    for kind, r0, c0, size in br.transpose_tiles(h):
        owner[r0:r0 + size, c0:c0 + size] += 1
        if kind == "offdiag":
            owner[c0:c0 + size, r0:r0 + size] += 1
    assert (owner == 1).all()


def test_resolve_threads_env(monkeypatch):
    monkeypatch.setenv("BITREV_THREADS", "3")
    assert br.resolve_threads() == 3
    assert br.resolve_threads(5) == 5
    monkeypatch.setenv("BITREV_THREADS", "0")
    with pytest.raises(ValueError):
        br.resolve_threads()


# --- recursion plan (reference tests/test_recursive.py:164-197) -----------


def test_trace_structure_even():
    trace = []
    rec._plan(0, 12, 0, br.RecursionPolicy(6), trace)
    kinds = [k for k, _, _ in trace]
    assert kinds.count("transpose") == 1
    assert kinds.count("base") == 2 * (1 << 6)
    t = kinds.index("transpose")
    assert t == 1 << 6


def test_trace_one_even_odd_per_odd_level():
    trace = []
    rec._plan(0, 11, 0, br.RecursionPolicy(4), trace)
    assert trace[0] == ("even_odd", 0, 11)
    assert sum(1 for k, _, w in trace if k == "even_odd" and w == 11) == 1


def test_first_odd_width():
    assert rec._first_odd_width(20, br.RecursionPolicy(9)) is None
    assert rec._first_odd_width(11, br.RecursionPolicy(4)) == 11
    assert rec._first_odd_width(26, br.RecursionPolicy(9)) == 13
    assert rec._first_odd_width(26, br.RecursionPolicy(9, 1)) is None


# --- schedules --------------------------------------------------------------


def test_swap_count_law():
    for b in range(1, 27):
        assert br.swap_count(b) == ((1 << b) - (1 << ((b + 1) // 2))) // 2
    assert len(br.cached_schedule(10)) == br.swap_count(10)
    with pytest.raises(ValueError):
        br.SwapSchedule(3, np.zeros((3, 3)))


def test_rev_naive_semantics():
    assert br.rev_naive(1, 3) == 4
    assert br.rev_naive(0b0110, 4) == 6
    assert [br.rev_naive(i, 3) for i in range(8)] == [0, 4, 2, 6, 1, 5, 3, 7]
    assert br.BYTE_TABLE[1] == 128 and br.BYTE_TABLE[255] == 255
    with pytest.raises(ValueError):
        br.rev_naive(8, 3)


def test_csv_round_trip(tmp_path):
    recs = [br.make_record("cobra", b, r, 1e-6 * (b + r) / 3) for b in (8, 9) for r in range(3)]
    p = tmp_path / "x.csv"
    br.write_csv(recs, p)
    assert br.read_csv(p) == recs
    assert p.read_text().splitlines()[0] == "method,b,n,replicate,elapsed_s,per_element_s"


# --- benchmark API (src/bench.py:69-110, 380-433) ----------------------------


def test_bench_config_defaults_match_reference_fields():
    cfg = br.BenchConfig()
    assert cfg.methods == br.METHOD_IDS and (cfg.b_min, cfg.b_max) == (8, 20)
    assert (cfg.replicates, cfg.warmup, cfg.element_kind) == (100, 3, "pair")
    assert cfg.memory_cap_bytes == 1 << 30 and cfg.unrolled_max_bits == 16
    br.validate_config(cfg)


@pytest.mark.parametrize("kw,frag", [
    ({"methods": ()}, "no methods"),
    ({"methods": ("cobra", "nope")}, "unknown methods"),
    ({"b_min": 9, "b_max": 8}, "b_min"),
    ({"replicates": 0}, "replicates"),
    ({"warmup": -1}, "warmup"),
    ({"element_kind": "c64"}, "element kind"),
    ({"cobra_q": -1}, "cobra_q"),
    ({"memory_cap_bytes": 0}, "memory_cap_bytes"),
    ({"base_bits": 0}, "base_bits"),
])
def test_bench_config_validation(kw, frag):
    with pytest.raises(ValueError, match=frag):
        br.validate_config(br.BenchConfig(**kw))


def test_tune_cobra_argument_checks():
    with pytest.raises(ValueError, match="must not be empty"):
        br.tune_cobra(10, [])
    with pytest.raises(ValueError, match="violate"):
        br.tune_cobra(10, [3, 6])
    with pytest.raises(ValueError, match="variant"):
        br.tune_cobra(10, [3], variant="stockham")
    with pytest.raises(ValueError, match="replicates"):
        br.tune_cobra(10, [3], replicates=0)


def test_gbs_sidecar(tmp_path):
    recs = [br.make_record("cobra", 20, r, 1e-5) for r in range(2)]
    p = tmp_path / "gbs.csv"
    br.write_gbs_sidecar(recs, p, "pair")
    rows = p.read_text().splitlines()
    assert rows[0] == "method,b,n,replicate,elem_bytes,bytes_moved,gb_per_s,gelem_per_s"
    f = rows[1].split(",")
    assert f[4] == "16" and int(f[5]) == 2 * (1 << 20) * 16
    assert abs(float(f[6]) - 2 * (1 << 20) * 16 / 1e-5 / 1e9) < 1e-6


def test_complete_schedule_is_lazy():
    s = br.cached_schedule(20)
    assert s.complete and len(s) == br.swap_count(20)
    assert s._pairs is None  # nothing materialised until .pairs is read
    e = br.SwapSchedule(3, np.array([[1, 4], [3, 6]]))
    assert not e.complete and len(e) == 2


def test_schedule_file_format(tmp_path):
    """save_schedule / load_schedule: the reference's BRSCHD01 layout
    (/root/reference/pkg/tests/test_schedule.py:135-167), on an explicit
    host schedule (generation needs the device)."""
    pairs = np.array([[2, 4], [1, 8], [3, 12], [5, 10], [7, 14], [11, 13]], dtype=np.int64)
    s = br.SwapSchedule(4, pairs)
    path = tmp_path / "s.bin"
    br.save_schedule(s, path)
    raw = path.read_bytes()
    assert raw[:8] == b"BRSCHD01" and raw[8] == 4 and len(raw) == 9 + 16 * 6
    back = br.load_schedule(path)
    assert back.b == 4 and np.array_equal(back.pairs, pairs) and not back.pairs.flags.writeable
    (tmp_path / "junk.bin").write_bytes(b"NOTMAGIC" + bytes([3]))
    with pytest.raises(ValueError, match="magic"):
        br.load_schedule(tmp_path / "junk.bin")
    (tmp_path / "cut.bin").write_bytes(raw[:-16])
    with pytest.raises(ValueError, match="expected"):
        br.load_schedule(tmp_path / "cut.bin")


def test_scalar_index_helpers():
    """rev_bytetable / count_leading_zeros / xor_next (src/bits.py:59-113),
    with the reference's known answers (pkg/tests/test_bits.py:137-142)."""
    assert br.xor_next(br.RevPair(0, 0), 3) == br.RevPair(1, 4)
    assert br.xor_next(br.RevPair(3, 6), 3) == br.RevPair(4, 1)
    rng = np.random.default_rng(7)
    for b in range(1, 49):
        for i in rng.integers(0, 1 << b, 20, dtype=np.uint64).tolist():
            assert br.rev_bytetable(int(i), b) == br.rev_naive(int(i), b)
    state = br.RevPair(0, 0)
    for i in range(1, 1 << 8):
        state = br.xor_next(state, 8)
        assert state == (i, br.rev_naive(i, 8))
    with pytest.raises(ValueError):
        br.xor_next(br.RevPair(255, 255), 8)
    assert br.count_leading_zeros(1) == 63 and br.count_leading_zeros(1 << 63) == 0
    with pytest.raises(ValueError):
        br.count_leading_zeros(0)
    with pytest.raises(ValueError):
        br.count_leading_zeros(1 << 64)
    with pytest.raises(ValueError):
        br.rev_bytetable(8, 3)


def test_every_reference_export_exists():
    """Drop-in: every name in the reference package's __all__
    (tests/golden/reference_exports.json, read from
    /root/reference/pkg/src/bitrev/__init__.py) is exported here too."""
    import json
    from pathlib import Path

    names = json.loads((Path(__file__).parent / "golden" / "reference_exports.json").read_text())["names"]
    missing = [n for n in names if not hasattr(br, n)]
    assert not missing, missing
    assert set(names) <= set(br.__all__)


def test_csv_edge_cases(tmp_path):
    """The reference's CSV contract (pkg/tests/test_bench.py:126-170): empty
    tables, trailing newline, header / short-row / inconsistent-n errors that
    name the file position, write failures that name the path."""
    p = tmp_path / "empty.csv"
    br.write_csv([], p)
    assert p.read_text() == "method,b,n,replicate,elapsed_s,per_element_s\n"
    assert br.read_csv(p) == []
    recs = [br.make_record("xor", 4, i, 1.5e-6 * (i + 1)) for i in range(3)]
    br.write_csv(recs, p)
    assert len(p.read_text().splitlines()) == 4 and p.read_text().endswith("\n")
    with pytest.raises(OSError, match="no/such/dir"):
        br.write_csv([], "no/such/dir/out.csv")
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(ValueError, match="header"):
        br.read_csv(bad)
    bad.write_text("method,b,n,replicate,elapsed_s,per_element_s\nxor,4,16,0\n")
    with pytest.raises(ValueError, match=":2"):
        br.read_csv(bad)
    bad.write_text("method,b,n,replicate,elapsed_s,per_element_s\nxor,4,99,0,1e-06,6.25e-08\n")
    with pytest.raises(ValueError, match="99"):
        br.read_csv(bad)
