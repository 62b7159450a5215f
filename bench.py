#!/usr/bin/env python
"""Benchmark: effective HBM GB/s (2*n*elem_bytes / time) of the bit-reversed
permutation on B200, plus the reference's CPU path timed on the host cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload W]
                    [--impl ours|reference]

A "step" is one permutation of one batch of synthetic input (BASELINE.json
configs).  BASELINE.json quotes its metric "vs log2 n" on no single config,
so the N=1 line is the largest single-GPU config: cfg3-16 = n=2^30 complex128
out of place (16 GiB per side); the same line carries cfg3-4 / cfg3-8 (the
element-width sweep of config 3) under "width_sweep", and the other configs
(cfg1, cfg2, cfg4, cfg4-fft7, cfg5's array on one GPU) under "other_configs",
each timed with the same protocol in the same run.  With N > 1 the default
is cfg5, the one config that shards a single array: n=2^32 complex64 split by
its top log2 N index bits, local reversal + NCCL all_to_all_single over
NVLink + local interleave, with per-phase times and all-to-all bus bandwidth.
The other configs are parity-test cases and --workload lines.

Timing: W untimed warm-up steps, then EXACTLY K steps timed with CUDA events
on the stream the kernel is launched on, with a barrier + device synchronise
on both sides; the job time is the max over ranks of the per-rank time.
Workloads whose working set is below 4x the L2 get an L2 flush (a 512 MiB
write) before every step, outside that step's own event pair, and the
per-rank time is the sum of the K step durations; the others (cfg3: 32 GiB
per step) exceed the L2 by two orders of magnitude and run their K steps back
to back between one event pair.

Under torchrun (N > 1) cfg1-cfg3 run one replica per rank ("replicas only":
a single array does not shard without an exchange), cfg4 shards the batch
rows (no collective), and cfg5 runs the top-bit sharded plan.  Rank 0 prints
ONE JSON line.

--impl reference times the reference's own CPU algorithm for the path on rank
0 with all host threads: the C restatement in oracle/ (parallel
semi-recursive, src/parallel.py:95-156) and, beside it, the reference package
itself (baseline/_ref, numba) on the same sample; the line's value is the
faster of the two.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (b, torch dtype name, elem bytes, in-place, batch, description)
    "cfg1": (20, "complex128", 16, False, 1,
             "out-of-place bit reversal, n=2^20 complex128 (parity target: recursive_permute)"),
    "cfg2": (26, "float64", 8, True, 1,
             "in-place bit reversal (tile-pair swap), n=2^26 float64"),
    "cfg3-4": (30, "float32", 4, False, 1, "out-of-place bit reversal, n=2^30 float32"),
    "cfg3-8": (30, "float64", 8, False, 1, "out-of-place bit reversal, n=2^30 float64"),
    "cfg3-16": (30, "complex128", 16, False, 1,
                "out-of-place bit reversal, n=2^30 complex128 (16 GiB per side; the largest "
                "single-GPU BASELINE config)"),
    "cfg4": (16, "complex64", 8, False, 4096,
             "batched out-of-place bit reversal, 4096 x n=2^16 complex64 (FFT pre-pass)"),
    "cfg4-fft7": (16, "complex64", 8, False, 4096,
                  "batched FFT pre-pass, 4096 x n=2^16 complex64: bit reversal fused with the "
                  "first 7 radix-2 DIT stages"),
    "cfg5": (32, "complex64", 8, False, 1,
             "n=2^32 complex64 sharded by top index bits: local reversal + NCCL "
             "all_to_all_single + interleave"),
}
METRIC = "effective HBM GB/s (2*n*elem_bytes/time)"
L2_BYTES = 126 * 10**6
FALLBACK_HBM_GBS = 6650.0
NVLINK_GBS_PER_DIRECTION = 900.0  # NVLink 5 through NVSwitch, per GPU per direction


def parse():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: cfg3-16 on one GPU, cfg5 (sharded) on N > 1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the cfg3 width sweep")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo + --same-device only to test the "
                         "multi-rank plumbing on one GPU)")
    ap.add_argument("--same-device", action="store_true",
                    help="debug: every rank uses cuda:0 (replica workloads only)")
    ap.add_argument("--tile-bits", type=int, default=0,
                    help="override the library's tile bits Q for this workload (tuning)")
    ap.add_argument("--tile-path", type=int, default=-1,
                    help="override the staging path (0 register, 1 bulk ring, 2 tensor ring, "
                         "3 rect [out of place], 4 cp.async / 5 TMA stores / 6 cluster "
                         "pairs [in place])")
    ap.add_argument("--chunks", type=int, default=4,
                    help="cfg5: all-to-all rounds (round c+1 on the wire while c is interleaved)")
    ap.add_argument("--p2p", action="store_true",
                    help="cfg5: time the fused scatter into peer-mapped symmetric memory as the "
                         "main line instead of NCCL")
    ap.add_argument("--no-fused", action="store_true",
                    help="cfg5, N > 1: skip the fused peer-store companion measurement")
    ap.add_argument("--no-soak", action="store_true",
                    help="skip the 0.5 s clock soak (for profiler runs)")
    ap.add_argument("--cpu-sample-s", type=float, default=10.0,
                    help="target seconds of CPU work for the cpu_baseline sample")
    ap.add_argument("--bits", type=int, default=0,
                    help="override the workload's log2 n (functional tests of the launch "
                         "plumbing at small sizes; never for reported numbers)")
    args = ap.parse_args()
    if args.workload is None:
        args.workload = default_workload(dist_env()[0])
    if args.bits:
        b, dt, E, ip, batch, desc = WORKLOADS[args.workload]
        WORKLOADS[args.workload] = (args.bits, dt, E, ip, batch,
                                    f"{desc} [TEST SIZE: n=2^{args.bits}]")
    return args


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def default_workload(world):
    """N=1: the largest single-GPU config (the BASELINE metric names no single
    config); N>1: the sharded single array, the config that scales across GPUs."""
    return "cfg3-16" if world == 1 else "cfg5"


def short_dtype(name):
    return {"float32": "f32", "float64": "f64", "complex64": "c64", "complex128": "c128"}[name]


# ---------------------------------------------------------------------------
# helpers


def load_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        v = float(json.loads(p.read_text())["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_traffic(workload):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture summary (profiles/traffic.json), or None."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text())[workload]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.marks = {}

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), line.strip()))

    def mark(self, name):
        self.marks[name] = time.monotonic()

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        def parse(rows):
            out = []
            for _, line in rows:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    out.append((float(f[0]), float(f[1]), f))
                except ValueError:
                    continue
            return out

        window = "timed"
        rows = parse([r for r in self.rows if t0 <= r[0] <= t1])
        if len(rows) < 3:  # timed region shorter than the sampling period
            window = "warmup+timed+soak"
            rows = parse([r for r in self.rows
                          if self.marks.get("load0", t0) <= r[0] <= self.marks.get("load1", t1)])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0, "window": "no nvidia-smi samples in the run"}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, f in rows:
            for k, name in enumerate(names):
                if f[4 + k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": sorted(reasons),
                "samples": len(rows), "window": window}


def host_info():
    info = {"logical_cpus": os.cpu_count()}
    try:
        import psutil

        info["physical_cores"] = psutil.cpu_count(logical=False)
        info["ram_gb"] = round(psutil.virtual_memory().total / 2**30, 1)
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return info


# ---------------------------------------------------------------------------
# the reference's CPU path (reference arm and cpu_baseline)


def load_reference_package():
    """The reference package itself, installed unmodified in baseline/_ref
    (pip install --target), or None when absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "bitrev" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/bitrev_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import bitrev  # noqa: F401  (the reference, not this repo's package)

        return bitrev
    except Exception as exc:  # numba missing or broken: report, time the port alone
        sys.stderr.write(f"reference package unavailable: {exc!r}\n")
        return None


NP_DTYPES = {"float32": np.float32, "float64": np.float64, "complex64": np.complex64,
             "complex128": np.complex128}


def _host_array(shape, np_dt):
    """A host array with every page touched (its values do not matter to a
    permutation's speed; a pattern fill is far cheaper than a random fill)."""
    a = np.empty(shape, dtype=np_dt)
    a.view(np.uint8).reshape(-1)[:] = 0x3F
    return a


def cpu_reference_runs(workload, threads):
    """The reference's CPU algorithm for the workload's path, as a list of
    (name, kind, step, bytes per step, sample, method): the C port (oracle/)
    and, when baseline/_ref is present, the reference package itself.  Both
    share one bounded host sample of the workload."""
    from oracle import oracle as orc

    orc.build()
    b, dtname, E, inplace, batch, _ = WORKLOADS[workload]
    np_dt = NP_DTYPES[dtname]
    ref = load_reference_package()
    runs = []
    if workload.startswith("cfg4"):
        # the reference has no batched API (and no FFT stages for cfg4-fft7:
        # its CPU path is the permutation alone): rows over a thread pool
        # created once; each step permutes a bounded block of rows
        import concurrent.futures as cf

        rows = max(threads, 64)
        arr = _host_array((rows, 1 << b), np_dt)
        out = np.empty_like(arr)
        pool = cf.ThreadPoolExecutor(threads)
        sample = f"{rows} of the {batch} rows per step"

        def port_step():
            list(pool.map(lambda r: orc.c_cobra_inplace(arr[r], b, 6), range(rows)))

        runs.append(("port", "port", port_step, 2 * rows * (1 << b) * E, sample,
                     "cobra_in_place (C port of src/permutations.py:252-321) per row, "
                     f"{threads}-thread pool"))
        if ref is not None:
            local = threading.local()

            def row(r):
                cfg = getattr(local, "cfg", None)
                if cfg is None:
                    cfg = local.cfg = ref.CobraConfig(6)
                ref.cobra_out_of_place(arr[r], out[r], cfg, b)

            def ref_step():
                list(pool.map(row, range(rows)))

            runs.append(("reference", "reference", ref_step, 2 * rows * (1 << b) * E, sample,
                         "bitrev.cobra_out_of_place (baseline/_ref, numba) per row, "
                         f"{threads}-thread pool"))
        return runs
    if workload == "cfg5":
        b = 28  # bounded sample: 2^28 of the 2^32 elements per step
    n = 1 << b
    arr = _host_array(n, np_dt)
    sample = (f"full n=2^{b} array per step" if workload != "cfg5" else
              "n=2^28 of the 2^32-element array per step")

    def port_step():
        orc.c_parallel_semi_recursive(arr, b, threads)

    runs.append(("port", "port", port_step, 2 * n * E, sample,
                 f"parallel_semi_recursive_permute (C port of src/parallel.py:95-156), "
                 f"{threads} threads"))
    if ref is not None:
        pcfg = ref.ParallelConfig(threads=threads)

        def ref_step():
            ref.parallel_semi_recursive_permute(arr, b, pcfg)

        runs.append(("reference", "reference", ref_step, 2 * n * E, sample,
                     f"bitrev.parallel_semi_recursive_permute (baseline/_ref, numba), "
                     f"{threads} threads"))
    return runs


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    runs = cpu_reference_runs(args.workload, threads)
    results = {}
    for name, kind, step, nbytes, sample, method in runs:
        for _ in range(max(args.warmup, 1)):  # the first call also JIT-compiles numba
            step()
        ts = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            step()
            ts.append(time.perf_counter() - t0)
        results[name] = {"value": nbytes * len(ts) / sum(ts) / 1e9, "unit": "GB/s",
                         "kind": kind, "ms_per_step": sum(ts) / len(ts) * 1e3,
                         "sample": sample, "method": method}
    best = max(results.values(), key=lambda r: r["value"])
    value = best["value"]
    b, dtname, E, inplace, batch, desc = WORKLOADS[args.workload]
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": best["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": short_dtype(dtname), "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.workload}: {desc}", "b": b, "elem_bytes": E,
                   "inplace": inplace, "batch": batch},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": best["kind"],
                         "sample": best["sample"], "method": best["method"],
                         "runs": results, "host": host_info()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def single_thread_methods(workload, budget_s=20.0):
    """The reference's single-thread methods on the same array.

    Up to 2 GiB per side: COBRA (q = default_cobra_q), semi-recursive and
    recursive through the C port, once each.  For config 3 (2^30 elements):
    the reference package's own cobra_out_of_place, the method BASELINE.md
    times at that size (src/permutations.py:293-308), once, after a small
    JIT warm-up.  GB/s."""
    from oracle import oracle as orc

    b, dtname, E, inplace, batch, _ = WORKLOADS[workload]
    np_dt = NP_DTYPES[dtname]
    if workload.startswith("cfg3"):
        ref = load_reference_package()
        if ref is None:
            return None
        small_a, small_d = _host_array(1 << 12, np_dt), np.empty(1 << 12, dtype=np_dt)
        ref.cobra_out_of_place(small_a, small_d, ref.CobraConfig(6), 12)  # JIT compile
        a = _host_array(1 << b, np_dt)
        d = np.empty_like(a)
        t0 = time.perf_counter()
        ref.cobra_out_of_place(a, d, ref.CobraConfig(6), b)
        dt = time.perf_counter() - t0
        return {"unit": "GB/s", "threads": 1, "kind": "reference",
                "values": {"cobra_out_of_place": round(2 * a.nbytes / dt / 1e9, 3)},
                "seconds": round(dt, 2)}
    if workload.startswith("cfg4") or workload == "cfg5" or (1 << b) * E > (2 << 30):
        return None
    a = _host_array(1 << b, np_dt)
    q = min(b // 2, 6)
    runs = [("cobra_in_place" if inplace else "cobra_out_of_place",
             (lambda: orc.c_cobra_inplace(a, b, q)) if inplace else (lambda: orc.c_cobra_oop(a, b, q))),
            ("semi_recursive_permute", lambda: orc.c_recursive(a, b, 9, 1)),
            ("recursive_permute", lambda: orc.c_recursive(a, b, 9, 0))]
    out = {}
    t_all = time.perf_counter()
    for name, fn in runs:
        if time.perf_counter() - t_all > budget_s:
            break
        t0 = time.perf_counter()
        fn()
        out[name] = round(2 * a.nbytes / (time.perf_counter() - t0) / 1e9, 3)
    return {"unit": "GB/s", "threads": 1, "values": out, "kind": "port"}


def cpu_baseline(workload, target_s):
    """The reference's CPU path timed on the host cores (the C port and the
    reference package itself), each bounded to ~target_s of CPU work."""
    threads = os.cpu_count() or 1
    runs = cpu_reference_runs(workload, threads)
    results = {}
    for name, kind, step, nbytes, sample, method in runs:
        t0 = time.perf_counter()
        step()  # warm (page faults, thread start-up, numba JIT)
        if time.perf_counter() - t0 < 2.0:  # first touches of a fresh sample run slow
            step()
            step()
        ts = []
        t_start = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            step()
            ts.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > target_s / threads or len(ts) >= 50:
                break
        results[name] = {"value": nbytes * len(ts) / sum(ts) / 1e9, "unit": "GB/s", "kind": kind,
                         "sample": f"{sample}, {len(ts)} steps", "method": method}
    best = max(results.values(), key=lambda r: r["value"])
    del runs
    gc.collect()
    return {"value": best["value"], "unit": "GB/s", "cores": threads, "kind": best["kind"],
            "sample": best["sample"], "method": best["method"], "runs": results,
            "host": host_info(), "single_thread": single_thread_methods(workload)}


# ---------------------------------------------------------------------------
# our arm


class Flush:
    """Write a 512 MiB buffer (evicts the inputs from the 126 MB L2), then read
    a 256 MiB one so the L2 is left holding clean lines: otherwise the timed
    kernel would pay for writing back the flush's own dirty lines."""

    def __init__(self, torch, dev):
        self.torch = torch
        self.w = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
        self.sink = torch.empty((), dtype=torch.float32, device=dev)

    def zero_(self):
        self.w.zero_()
        self.torch.sum(self.r, dim=0, out=self.sink)


def kernel_family(chosen, inplace):
    """Kernel family of a (tile bits, staging path) choice (bitrev_last_tile)."""
    path = chosen[1]
    if path == 1:
        return f"bitrev_ring_kernel (TMA bulk-row ring, Q={chosen[0]})"
    if path == 2:
        return f"bitrev_ring_kernel (TMA tensor-map ring, Q={chosen[0]})"
    if path == 3:
        return f"bitrev_oop_rect_kernel (QX={chosen[0]})"
    if path == 6:
        return f"bitrev_inplace_cluster_kernel (Q={chosen[0]})"
    if path == -3:
        return "bitrev_rows_kernel (short rows)"
    if inplace:
        return f"bitrev_inplace_tile_kernel (Q={chosen[0]})"
    return f"bitrev_oop_tile_kernel (Q={chosen[0]})"


def time_steps(torch, step, steps, stream, flush=None):
    """Per-step seconds of `steps` steps timed with CUDA events on `stream`.

    Without a flush the K steps run back to back between ONE event pair and
    each step is credited K-th of the span (an event record between steps
    costs ~3 us of device time, 2 % of cfg2's 181 us step:
    tools/event_overhead_probe.py).  With an L2 flush every step has its own
    event pair and the flush stays outside it."""
    if flush is None:
        s0 = torch.cuda.Event(enable_timing=True)
        e0 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(steps):
            step()
        e0.record(stream)
        torch.cuda.synchronize()
        return [s0.elapsed_time(e0) / 1e3 / steps] * steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for k in range(steps):
        if flush is not None:
            flush.zero_()
        starts[k].record(stream)
        step()
        ends[k].record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) / 1e3 for s, e in zip(starts, ends)]


def plain_step(wl, x, y, stream):
    """The device step of a single-GPU workload on resident buffers x (, y)."""
    from paper_1708_01873_b200 import _core, _lib

    b, _, E, inplace, _, _ = WORKLOADS[wl]
    if wl == "cfg4-fft7":
        rows = x.shape[0]
        return lambda: _lib.call("bitrev_dit_prepass", x.data_ptr(), y.data_ptr(), b, E, rows,
                                 1 << b, 1 << b, 7, 0, stream.cuda_stream)
    if inplace:
        return lambda: _core.launch_inplace(x, b)
    return lambda: _core.launch_oop(x, y, b)


def config_sweep(torch, dev, peak, steps, workloads):
    """The other BASELINE configs on the same device in the same run, each
    with the main line's protocol (L2 flush before every step below 4x the
    L2, CUDA events per step, W = 3 warm-up steps), fewer steps; cfg5 is its
    whole 2^32-element array on this one GPU."""
    from paper_1708_01873_b200 import _lib

    out = {}
    stream = torch.cuda.current_stream(dev)
    for w in workloads:
        b, dtname, E, inplace, batch, desc = WORKLOADS[w]
        shape = (batch, 1 << b) if batch > 1 else (1 << b,)
        n = batch << b
        x = torch.empty(n * E, dtype=torch.uint8, device=dev).random_(0, 256)
        x = x.view(getattr(torch, dtname)).view(shape)
        y = None if inplace else torch.empty_like(x)
        step = plain_step(w, x, y, stream)
        nbytes = 2 * n * E
        flush = Flush(torch, dev) if nbytes < 4 * L2_BYTES else None
        for _ in range(5):
            if flush is not None:
                flush.zero_()
            step()
        torch.cuda.synchronize()
        ts = time_steps(torch, step, steps, stream, flush)
        v = nbytes * len(ts) / sum(ts) / 1e9
        q, path = _lib.last_tile()
        out[w] = {"value": v, "unit": "GB/s", "gelem_per_s": v / (2 * E), "frac": v / peak,
                  "ms_per_step": sum(ts) / len(ts) * 1e3,
                  "median_ms": statistics.median(ts) * 1e3, "steps": steps,
                  "step_ms_all": [round(t * 1e3, 4) for t in ts],
                  "tile_bits": None if w == "cfg4-fft7" else q,
                  "tile_path": None if w == "cfg4-fft7" else path,
                  "kernel": ("bitrev_fft_rect_kernel" if w == "cfg4-fft7" else
                             kernel_family((q, path), inplace)),
                  "l2": "flushed before every step" if flush else "inputs larger than L2, no flush",
                  "workload": desc}
        del x, y, flush
        gc.collect()
        torch.cuda.empty_cache()
    return out


def e2e_host(torch, br, x, b, E, inplace, workload, steps, stream):
    """End to end through the public API with host buffers (rank 0's replica).

    e2e: bitrev_host_pipeline (cfg4-fft7: dit_prepass_host_pipeline) over a
    stream of pinned host arrays (each step = one array: its H2D copy, the
    kernel and its D2H copy; consecutive steps overlap their copies in
    opposite directions).  e2e_single: one
    blocking reference-style call per array (cobra_in_place /
    cobra_out_of_place / bitrev_batched / bitrev_dit_prepass on a host tensor:
    H2D, kernel, D2H, sync, nothing overlapped).  All host buffers are freed
    before returning."""
    n_local = x.numel()
    bytes_local = 2 * n_local * E
    nhost = 3
    hosts = [x.cpu().pin_memory() for _ in range(nhost)]
    houts = None if inplace else [torch.empty_like(h).pin_memory() for h in hosts]
    cfg = br.CobraConfig(6)
    # arrays streamed through the pipeline: its first H2D and last D2H have
    # no opposite-direction copy to overlap, so the per-step figure
    # approaches the steady state as 1 - ~1/reps (48: within ~2 %)
    reps = min(64, max(48, steps))
    e2e = e2e_single = None

    def run_pipeline():
        srcs = [hosts[k % nhost] for k in range(reps)]
        dsts = None if houts is None else [houts[k % nhost] for k in range(reps)]
        if workload == "cfg4-fft7":
            br.dit_prepass_host_pipeline(srcs, b, 7, dsts)
        else:
            br.bitrev_host_pipeline(srcs, b, dsts)

    def single_step():
        if workload == "cfg4-fft7":
            br.bitrev_dit_prepass(hosts[0], b, 7, out=houts[0])
        elif workload == "cfg4":
            br.bitrev_batched(hosts[0], b, houts[0])
        elif inplace:
            br.cobra_in_place(hosts[0], cfg, b)
        else:
            br.cobra_out_of_place(hosts[0], houts[0], cfg, b)

    plan = ((run_pipeline, reps, "pipe"), (single_step, 1, "single"))
    for fn, n_steps, key in plan:
        fn()  # warm (stream/pool creation, page-locking caches)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        loops = 1 if key == "pipe" else min(reps, 5)
        ev0.record(stream)
        for _ in range(loops):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        t_step = ev0.elapsed_time(ev1) / 1e3 / (n_steps * loops)
        rec = {"value": bytes_local / t_step / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": n_local * E, "d2h_bytes_per_step": n_local * E,
               "ms_per_step": t_step * 1e3}
        if key == "pipe":
            api = ("dit_prepass_host_pipeline" if workload == "cfg4-fft7" else
                   "bitrev_host_pipeline")
            rec["path"] = (f"{api} over {reps} pinned host arrays (public API; per step: "
                           "H2D + kernel + D2H, consecutive steps overlapped)")
            e2e = rec
        else:
            rec["path"] = ("one blocking call per array on a pinned host tensor "
                           "(cobra_in_place / cobra_out_of_place / bitrev_batched / "
                           "bitrev_dit_prepass)")
            e2e_single = rec
    if e2e is None:
        e2e = e2e_single
    else:
        # PCIe ceiling for the pipeline, same harness: each step one H2D and one
        # D2H of the step's bytes, both split into 256 MiB pieces over two
        # streams per direction exactly like the pipeline's copies, no kernel.
        d_in, d_out = torch.empty_like(x), torch.empty_like(x)
        h_out = houts if houts is not None else hosts
        ups = [torch.cuda.Stream(), torch.cuda.Stream()]
        downs = [torch.cuda.Stream(), torch.cuda.Stream()]
        chunk = (256 << 20) // x.element_size()
        fd_in, fd_out = d_in.view(-1), d_out.view(-1)
        for timed in (False, True):
            torch.cuda.synchronize()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for st_ in ups + downs:
                st_.wait_stream(stream)
            for k in range(reps if timed else 2):
                src_h = hosts[k % nhost].view(-1)
                dst_h = h_out[(k + 1) % nhost].view(-1)
                for i, o in enumerate(range(0, fd_in.numel(), chunk)):
                    with torch.cuda.stream(ups[i & 1]):
                        fd_in[o:o + chunk].copy_(src_h[o:o + chunk], non_blocking=True)
                    with torch.cuda.stream(downs[i & 1]):
                        dst_h[o:o + chunk].copy_(fd_out[o:o + chunk], non_blocking=True)
            for st_ in ups + downs:
                stream.wait_stream(st_)
            ev1.record(stream)
            torch.cuda.synchronize()
        ceil = bytes_local / (ev0.elapsed_time(ev1) / 1e3 / reps) / 1e9
        e2e["pcie_ceiling_gbs"] = ceil
        e2e["frac_of_pcie_ceiling"] = e2e["value"] / ceil
        e2e["pcie_ceiling_path"] = ("concurrent pinned H2D + D2H of the step's bytes, each "
                                    "as 256 MiB pieces over two streams per direction, no "
                                    "kernel (same harness)")
        del d_in, d_out
    del hosts, houts
    gc.collect()
    torch.cuda.empty_cache()
    return e2e, e2e_single


def e2e_sharded(torch, dist, sharded, x, b, chunks, steps, stream, world):
    """cfg5 end to end through sharded_bitrev: every rank copies its shard in
    from pinned host memory, runs the sharded permutation, and copies its
    output shard back; max over ranks."""
    E = x.element_size()
    host_in = x.cpu().pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    dev_in = torch.empty_like(x)

    def step():
        dev_in.copy_(host_in, non_blocking=True)
        out = sharded.sharded_bitrev(dev_in, b, chunks=chunks)
        host_out.copy_(out, non_blocking=True)

    step()
    torch.cuda.synchronize()
    reps = max(3, min(steps, 5))
    dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(reps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([ev0.elapsed_time(ev1) / 1e3 / reps], dtype=torch.float64, device=x.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t.item())
    rec = {"value": (1 << b) * 2 * E / t_step / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": x.numel() * E, "d2h_bytes_per_step": x.numel() * E,
           "bytes_are": "per rank (each rank moves its own shard)", "ms_per_step": t_step * 1e3,
           "path": "per rank: pinned H2D of the shard, sharded_bitrev (pack, all_to_all_single "
                   "rounds, unpack), D2H of the output shard; max over ranks"}
    del host_in, host_out, dev_in
    gc.collect()
    torch.cuda.empty_cache()
    return rec


def cfg5_phases(torch, dist, sharded, x, b, world, reps=3):
    """Per-phase device times of the sharded plan with one exchange round
    (pack -> all_to_all_single -> unpack), median of `reps`, max over ranks."""
    names = ("pack", "a2a", "unpack")
    acc = {k: [] for k in names}
    for _ in range(reps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ph = {}
        sharded.sharded_bitrev(x, b, chunks=1, phases=ph)
        torch.cuda.synchronize()
        acc["pack"].append(ph["t0"].elapsed_time(ph["packed"]) / 1e3)
        acc["a2a"].append(ph["packed"].elapsed_time(ph["exchanged"]) / 1e3)
        acc["unpack"].append(ph["exchanged"].elapsed_time(ph["done"]) / 1e3)
    med = torch.tensor([statistics.median(acc[k]) for k in names], dtype=torch.float64,
                       device=x.device)
    if world > 1:
        dist.all_reduce(med, op=dist.ReduceOp.MAX)
    t = dict(zip(names, med.tolist()))
    S = x.numel() * x.element_size()  # per-rank shard bytes
    out = {"ms": {k: v * 1e3 for k, v in t.items()}, "shard_bytes": S,
           "method": f"CUDA events on the current stream, one round, median of {reps}, max over ranks"}
    if world > 1 and t["a2a"] > 0:
        algbw = S / t["a2a"] / 1e9
        busbw = algbw * (world - 1) / world
        out["a2a"] = {"algbw_gbs": algbw, "busbw_gbs": busbw,
                      "peak_gbs_per_direction": NVLINK_GBS_PER_DIRECTION,
                      "frac_of_nvlink": busbw / NVLINK_GBS_PER_DIRECTION,
                      "convention": "nccl-tests: algbw = shard bytes / time, "
                                    "busbw = algbw * (G-1)/G"}
    if t["pack"] > 0:
        out["pack_hbm_gbs"] = 2 * S / t["pack"] / 1e9
    if t["unpack"] > 0 and world > 1:
        out["unpack_hbm_gbs"] = 2 * S / t["unpack"] / 1e9
    return out


def fused_p2p_companion(torch, dist, sharded, x, b, rank, world, steps, stream):
    """cfg5 at N > 1: the fused local-reversal + peer-store exchange
    (sharded_bitrev_p2p over torch symmetric memory) beside the NCCL line.
    Every rank must set up its peer views (agreed by an all-reduce), the
    fused result must equal the NCCL result byte for byte on every rank, and
    only then is it timed (CUDA events per step, max over ranks).  Any failure
    is reported in the returned record instead of the value."""
    ok, why = 1, ""
    try:
        peers, barrier, keep = sharded.symmetric_recv(x.numel(), x.dtype, x.device)
    except Exception as exc:  # no symmetric memory / peer mapping on this node
        ok, why = 0, f"{type(exc).__name__}: {exc}"[:300]
    flag = torch.tensor([ok], dtype=torch.int32, device=x.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if not int(flag.item()):
        return {"value": None, "error": why or "peer views unavailable on another rank"}
    ref = sharded.sharded_bitrev(x, b, chunks=1)
    got = sharded.sharded_bitrev_p2p(x, b, peers, rank, barrier)
    same = torch.tensor([int(torch.equal(ref.view(torch.uint8), got.view(torch.uint8)))],
                        dtype=torch.int32, device=x.device)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    del ref, got
    if not int(same.item()):
        return {"value": None, "error": "fused result differs from the NCCL result"}
    step = lambda: sharded.sharded_bitrev_p2p(x, b, peers, rank, barrier)  # noqa: E731
    for _ in range(3):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    ts = time_steps(torch, step, steps, stream)
    t = torch.tensor([sum(ts)], dtype=torch.float64, device=x.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    job = float(t.item())
    E = x.element_size()
    del keep
    return {"value": (1 << b) * 2 * E * steps / job / 1e9, "unit": "GB/s",
            "ms_per_step": job / steps * 1e3, "steps": steps,
            "path": "bitrev_sharded_scatter (rectangular tiles stored into the peers' "
                    "symmetric-memory receive buffers over NVLink), barrier, unpack, barrier",
            "checked": "byte-equal to the NCCL result on every rank"}


FUSED_TIMEOUT_S = 240.0


def guarded_fused_companion(torch, dist, sharded, x, b, rank, world, steps, stream, line):
    """fused_p2p_companion under a watchdog.  The companion is the only step
    that allocates symmetric memory and maps peers; if that stalls on some
    node (a rendezvous that never completes), every rank's timer fires after
    FUSED_TIMEOUT_S: rank 0 prints the finished line with the companion
    marked as timed out, and every rank exits 0, so the NCCL measurement is
    never lost to the companion."""
    lock = threading.Lock()
    state = {"done": False}

    def on_timeout():
        with lock:
            if state["done"]:
                return
            state["done"] = True
            if rank == 0:
                line["fused_p2p"] = {"value": None,
                                     "error": f"timed out after {FUSED_TIMEOUT_S:.0f} s"}
                print(json.dumps(line), flush=True)
            sys.stderr.flush()
            os._exit(0)

    timer = threading.Timer(FUSED_TIMEOUT_S, on_timeout)
    timer.daemon = True
    gc.collect()
    torch.cuda.empty_cache()  # the symmetric heap is a separate allocation
    timer.start()
    try:
        rec = fused_p2p_companion(torch, dist, sharded, x, b, rank, world, steps, stream)
    except Exception as exc:  # report, keep the line
        rec = {"value": None, "error": f"{type(exc).__name__}: {exc}"[:300]}
    with lock:
        if state["done"]:  # the watchdog already printed and is exiting
            time.sleep(3600)
        state["done"] = True
    timer.cancel()
    gc.collect()
    torch.cuda.empty_cache()
    return rec


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_1708_01873_b200 as br
    from paper_1708_01873_b200 import _core, _lib, sharded

    world, rank, local = dist_env()
    if world > 1:
        dev_index = 0 if args.same_device else local
        torch.cuda.set_device(dev_index)
        if args.dist_backend == "nccl":
            # NCCL's init lines (rank / nranks / transport) go to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", torch.cuda.current_device())
    b, dtname, E, inplace, batch, desc = WORKLOADS[args.workload]
    dtype = getattr(torch, dtname)
    peak, peak_src = load_peak()

    # per-rank work
    if args.workload.startswith("cfg4"):
        rows = batch // world
        scaling = "strong"
        shape = (rows, 1 << b)
    elif args.workload == "cfg5":
        g = sharded.check_plan(b, world)
        shape = (1 << (b - g),)
        scaling = "strong"
    else:
        shape = (1 << b,)
        scaling = "weak"
    n_local = int(np.prod(shape))
    bytes_local = 2 * n_local * E

    x = torch.empty(n_local * E, dtype=torch.uint8, device=dev).random_(0, 256).view(dtype)
    x = x.view(shape)
    y = None if (inplace or args.workload == "cfg5") else torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    if args.tile_bits:
        _lib.set_tile_bits(E, inplace, args.tile_bits)
    if args.tile_path >= 0:
        _lib.set_tile_path(E, inplace, args.tile_path)
    exchange = None
    if args.workload == "cfg5":
        exchange = (f"NCCL all_to_all_single in {args.chunks} rounds, round c interleaved while "
                    "c+1.. are on the wire" if world > 1 else "none (one GPU holds the array)")
        chunks = args.chunks if world > 1 else 1
        if args.p2p and world > 1:
            try:
                peers, p2p_barrier, _keep = sharded.symmetric_recv(n_local, dtype, dev)
                exchange = "fused scatter into symmetric memory (NVLink peer stores)"

                def step():
                    return sharded.sharded_bitrev_p2p(x, b, peers, rank, p2p_barrier)
            except Exception as exc:  # no peer mapping available: report and use NCCL
                exchange = f"{exchange} (p2p unavailable: {type(exc).__name__})"
                args.p2p = False
        if not (args.p2p and world > 1):
            def step():
                return sharded.sharded_bitrev(x, b, chunks=chunks)
    else:
        step = plain_step(args.workload, x, y, stream)

    need_flush = 2 * bytes_local < 4 * L2_BYTES and args.workload != "cfg5"
    flush = Flush(torch, dev) if need_flush else None

    sampler = ClockSampler(dev.index)
    sampler.start()
    sampler.mark("load0")
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # clock soak: keep the GPU busy >= 0.5 s and until nvidia-smi (slow to
    # start) has delivered a few samples under load (bounded at 5 s)
    t_soak = time.monotonic()
    while not args.no_soak and time.monotonic() - t_soak < 5.0 and (
            time.monotonic() - t_soak < 0.5 or len(sampler.rows) < 3):
        for _ in range(8):
            if flush is not None:
                flush.zero_()
            step()
        torch.cuda.synchronize()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    t_wall0 = time.monotonic()
    step_s = time_steps(torch, step, args.steps, stream, flush)
    t_wall1 = time.monotonic()
    launches = _lib.launch_count() - launches0
    chosen = _lib.last_tile()  # (tile bits, staging path) the timed launches used
    if world > 1:
        dist.barrier()
    rank_time = sum(step_s)
    if world > 1:
        t = torch.tensor([rank_time], dtype=torch.float64,
                         device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        job_time = float(t.item())
    else:
        job_time = rank_time
    sampler.mark("load1")

    # cfg5: per-phase times and all-to-all bandwidth (one round, instrumented)
    phases = None
    if args.workload == "cfg5" and not args.p2p:
        phases = cfg5_phases(torch, dist, sharded, x, b, world)

    # same-harness reference: torch copy_ of the same bytes with the same
    # flush protocol (a device copy moves 2*n*E bytes, like one permutation)
    copy_ref = None
    if args.workload != "cfg5":
        cdst = y if y is not None else torch.empty_like(x)
        cts = []
        for k in range(max(5, min(args.steps, 20))):
            if flush is not None:
                flush.zero_()
            c0 = torch.cuda.Event(enable_timing=True)
            c1 = torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            cdst.copy_(x)
            c1.record(stream)
            c1.synchronize()
            cts.append(c0.elapsed_time(c1) / 1e3)
        cts.sort()
        copy_ref = bytes_local / cts[len(cts) // 2] / 1e9
        del cdst

    # L2-hot companion for the flushed (L2-sized) workloads, SURVEY 8(d) d2:
    # 20 steps captured in one CUDA graph (launch latency amortised) and
    # replayed back to back with no flush, so the working set stays in L2.
    # Reported beside `value`, which stays the L2-flushed figure.
    l2_hot = None
    if need_flush:
        reps_per_graph, replays = 20, 5
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()  # warm on the capture stream
        stream.wait_stream(side)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph):
            for _ in range(reps_per_graph):
                step()
        graph.replay()
        torch.cuda.synchronize()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(replays):
            graph.replay()
        h1.record(stream)
        torch.cuda.synchronize()
        t_launch = h0.elapsed_time(h1) / 1e3 / (replays * reps_per_graph)
        l2_hot = {"value": bytes_local / t_launch / 1e9, "unit": "GB/s",
                  "us_per_launch": t_launch * 1e6,
                  "method": f"CUDA graph of {reps_per_graph} launches replayed {replays}x, "
                            "no L2 flush (working set L2-resident)"}
        del graph

    e2e = e2e_single = None
    if not args.no_e2e:
        if args.workload == "cfg5":
            if world > 1 and not args.p2p:
                e2e = e2e_sharded(torch, dist, sharded, x, b, args.chunks, args.steps, stream, world)
        elif rank == 0:
            e2e, e2e_single = e2e_host(torch, br, x, b, E, inplace, args.workload, args.steps,
                                       stream)
    sweep = others = None
    if args.workload == "cfg3-16" and not args.no_sweep and world == 1:
        del x, y
        x = y = None
        gc.collect()
        torch.cuda.empty_cache()
        sweep = config_sweep(torch, dev, peak, max(5, min(args.steps, 10)), ("cfg3-4", "cfg3-8"))
        others = config_sweep(torch, dev, peak, max(10, args.steps),
                              ("cfg1", "cfg2", "cfg4", "cfg4-fft7", "cfg5"))
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)

    if world > 1:
        dist.barrier()

    avg_launch = statistics.mean(step_s)
    achieved = bytes_local / avg_launch / 1e9
    value = world * bytes_local * args.steps / job_time / 1e9
    if args.workload == "cfg5":
        value = (1 << b) * 2 * E * args.steps / job_time / 1e9
    traffic = load_traffic(args.workload)
    kernel = ("bitrev_fft_rect_kernel" if args.workload == "cfg4-fft7" else
              kernel_family(chosen, inplace))
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": job_time / args.steps * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": short_dtype(dtname), "data": "synthetic (random bit patterns, device-generated)",
        "config": {
            "workload": f"{args.workload}: {desc}", "b": b, "elem_bytes": E, "inplace": inplace,
            "batch": batch, "per_gpu_bytes_moved": bytes_local,
            "parallelism": {"cfg4": f"batch rows sharded over {world} GPUs",
                            "cfg4-fft7": f"batch rows sharded over {world} GPUs",
                            "cfg5": f"top {world.bit_length() - 1} index bits over {world} GPUs"
                            }.get(args.workload, f"replicas only ({world} independent arrays)"),
            "l2": "L2 flushed before every step (512 MiB write, then a 256 MiB read so "
                  "no dirty flush lines remain), outside the step's events" if need_flush else
                  f"inputs larger than L2 ({bytes_local // 2 >> 20} MiB per side per rank), "
                  "no flush",
            "tile_bits": None if args.workload == "cfg4-fft7" else chosen[0],
            "tile_path": None if args.workload == "cfg4-fft7" else chosen[1],
        },
        "gelem_per_s": value / (2 * E),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": kernel,
                     "algorithmic_bytes_per_launch": bytes_local, "peak_source": peak_src,
                     "frac_of_8TBs_spec": achieved / 8000.0,
                     "torch_copy_same_harness_gbs": copy_ref,
                     "frac_of_torch_copy_same_harness": (achieved / copy_ref) if copy_ref else None},
        "e2e": e2e,
        "e2e_single_call": e2e_single,
        "l2_hot": l2_hot,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "step_ms": {"median": statistics.median(step_s) * 1e3, "min": min(step_s) * 1e3,
                    "max": max(step_s) * 1e3, "all": [round(t * 1e3, 4) for t in step_s],
                    "method": ("one event pair around the K back-to-back steps"
                               if flush is None else
                               "an event pair per step, the L2 flush outside it")},
    }
    if sweep is not None:
        line["width_sweep"] = sweep
    if others is not None:
        line["other_configs"] = others
    if args.workload == "cfg5":
        line["config"]["exchange"] = exchange
        line["config"]["chunks"] = args.chunks if world > 1 else 1
        if world > 1:
            # the step is NVLink-bound; the HBM roofline applies to the local passes
            line["roofline"]["kernel"] = "local pack (bitrev_sharded_pack) + unpack"
            line["roofline"]["achieved_note"] = ("per-rank step bytes 2*S / step time "
                                                 "(all three phases)")
            if phases and "a2a" in phases:
                line["nvlink_roofline"] = phases["a2a"]
        else:
            line["roofline"]["kernel"] = f"{kernel} (2^32 elements on one GPU)"
        if phases is not None:
            line["phases"] = phases
    if (args.workload == "cfg5" and not args.p2p and world > 1 and args.dist_backend == "nccl"
            and not args.no_fused):
        # last, because it is the one step that maps peer memory: a watchdog
        # prints the line without it if the symmetric-memory setup stalls
        line["fused_p2p"] = guarded_fused_companion(
            torch, dist, sharded, x, b, rank, world, max(3, min(args.steps, 10)), stream, line)
    if rank != 0:
        dist.destroy_process_group()
        return 0
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.workload, args.cpu_sample_s)
        except Exception as e:  # keep the GPU line even if the host port fails
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
