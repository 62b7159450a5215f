"""bench.py's multi-rank launch plumbing.

* CPU: the reference arm under torchrun with two ranks -- rank 0 times the
  reference's CPU path and prints exactly one JSON line, rank 1 exits 0
  without work (the driver launches both arms the same way).
* GPU (one device): cfg4 under torchrun with two ranks on the same GPU over
  gloo.  cfg4 shards batch rows with no data-path collective, so the ranks'
  kernels never wait on one another; this checks the barrier / max-over-ranks
  / one-line plumbing, not multi-GPU performance.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, timeout):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           *args]
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def _json_lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def test_reference_arm_two_ranks():
    p = _torchrun(["--impl", "reference", "--gpus", "2", "--workload", "cfg1", "--steps", "2",
                   "--warmup", "1"], timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1, p.stdout[-2000:]
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_cfg4_two_ranks_one_device(cuda):
    p = _torchrun(["--gpus", "2", "--workload", "cfg4", "--steps", "3", "--warmup", "3",
                   "--same-device", "--dist-backend", "gloo", "--no-e2e", "--no-soak"],
                  timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1, p.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] == 3
    assert d["config"]["parallelism"] == "batch rows sharded over 2 GPUs"
    assert d["config"]["per_gpu_bytes_moved"] == 2 * 2048 * (1 << 16) * 8


@pytest.mark.gpu
def test_cfg5_two_ranks_one_device_gloo(cuda):
    """cfg5's N > 1 bench path (pack, all_to_all_single rounds, unpack, the
    per-phase instrumented round, the host-buffer e2e, max over ranks) at a
    test size, two ranks on one device over gloo: a functional check of the
    line the SCALE runs print, not a timing."""
    p = _torchrun(["--gpus", "2", "--workload", "cfg5", "--bits", "24", "--steps", "3",
                   "--warmup", "3", "--same-device", "--dist-backend", "gloo", "--no-soak"],
                  timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1, p.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["config"]["chunks"] == 4 and "all_to_all_single" in d["config"]["exchange"]
    assert set(d["phases"]["ms"]) == {"pack", "a2a", "unpack"}
    assert d["nvlink_roofline"]["busbw_gbs"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == (1 << 23) * 8
    assert d["gpu_launches"] == 3 * (1 + 4)  # per step: one pack, one unpack per round
    assert "TEST SIZE" in d["config"]["workload"]


_WATCHDOG = r"""
import json, sys, time
sys.path.insert(0, {root!r})
import torch
import bench
bench.FUSED_TIMEOUT_S = {timeout}
def companion(*a):
    time.sleep({sleep})
    return {{"value": 1.0}}
bench.fused_p2p_companion = companion
line = {{"metric": "m", "value": 2.0}}
rec = bench.guarded_fused_companion(torch, None, None, None, 0, 0, 2, 3, None, line)
print("RETURNED", json.dumps(rec))
"""


def _watchdog_run(timeout, sleep):
    code = _WATCHDOG.format(root=str(ROOT), timeout=timeout, sleep=sleep)
    return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                          timeout=120)


def test_fused_companion_watchdog_prints_line_and_exits_0():
    """A stalled peer-memory setup must not cost the cfg5 line: rank 0's
    watchdog prints the finished line (companion marked timed out) and the
    process exits 0."""
    p = _watchdog_run(timeout=0.5, sleep=30)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1 and "RETURNED" not in p.stdout
    assert lines[0]["value"] == 2.0
    assert lines[0]["fused_p2p"]["value"] is None
    assert "timed out" in lines[0]["fused_p2p"]["error"]


def test_fused_companion_watchdog_quiet_when_in_time():
    p = _watchdog_run(timeout=30, sleep=0)
    assert p.returncode == 0, p.stderr[-2000:]
    assert _json_lines(p.stdout) == []
    assert 'RETURNED {"value": 1.0}' in p.stdout


def test_kernel_family_names_the_launch():
    """bench.py labels roofline.kernel from the launch's (tile bits, path)."""
    sys.path.insert(0, str(ROOT))
    import bench

    assert bench.kernel_family((6, 0), False) == "bitrev_oop_tile_kernel (Q=6)"
    assert bench.kernel_family((7, 3), False) == "bitrev_oop_rect_kernel (QX=7)"
    assert bench.kernel_family((4, 2), False).startswith("bitrev_ring_kernel (TMA tensor-map")
    assert bench.kernel_family((6, 1), False).startswith("bitrev_ring_kernel (TMA bulk-row")
    assert bench.kernel_family((6, 0), True) == "bitrev_inplace_tile_kernel (Q=6)"
    assert bench.kernel_family((6, 6), True) == "bitrev_inplace_cluster_kernel (Q=6)"
    assert bench.kernel_family((0, -3), False) == "bitrev_rows_kernel (short rows)"
