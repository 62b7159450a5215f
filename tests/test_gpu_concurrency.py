"""Concurrent calls on distinct arrays are safe (the reference's nogil
contract): several host threads, each on its own CUDA
stream and arrays, call the in-place, out-of-place and host-staged entry
points at once (ctypes releases the GIL).  Every result is byte-compared with
the oracle, and every thread's bitrev_last_tile reports its own launches.
"""

import threading

import numpy as np
import pytest
import torch

import paper_1708_01873_b200 as br
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _worker(idx, cuda, errors, rounds=12):
    try:
        rng = np.random.default_rng(100 + idx)
        stream = torch.cuda.Stream(cuda)
        E, dt = [(4, np.int32), (8, np.int64), (16, np.complex128), (8, np.float64)][idx % 4]
        for r in range(rounds):
            b = 14 + (r + idx) % 9  # 14..22: whole-row, mid-size and large tiles
            host = rng.integers(0, 256, (1 << b) * E, dtype=np.uint8).view(dt)
            want = orc.oracle_permute(host, b).view(np.uint8)
            with torch.cuda.stream(stream):
                a = torch.from_numpy(host).to(cuda, non_blocking=False)
                out = torch.empty_like(a)
                br.cobra_out_of_place(a, out, br.CobraConfig(0), b)
                q_oop = br.last_tile()
                br.cobra_in_place(a, br.CobraConfig(0), b)
                stream.synchronize()
            if not np.array_equal(out.cpu().numpy().view(np.uint8), want):
                errors.append(f"thread {idx} b={b}: out of place differs")
            if not np.array_equal(a.cpu().numpy().view(np.uint8), want):
                errors.append(f"thread {idx} b={b}: in place differs")
            if q_oop[1] == -2:  # 4/8/16-byte aligned arrays never need the element-wise kernel
                errors.append(f"thread {idx} b={b}: unexpected element-wise launch")
            h = host.copy()
            br.cobra_in_place(h, br.CobraConfig(0), b)  # numpy: host-staged, synchronous
            if not np.array_equal(h.view(np.uint8), want):
                errors.append(f"thread {idx} b={b}: host-staged call differs")
    except Exception as exc:  # surface any exception from the thread
        errors.append(f"thread {idx}: {type(exc).__name__}: {exc}")


@pytest.mark.parametrize("threads", [4])
def test_concurrent_calls_on_distinct_arrays(cuda, threads):
    errors = []
    ts = [threading.Thread(target=_worker, args=(i, cuda, errors)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "a worker thread hung"
    assert not errors, errors[:5]
