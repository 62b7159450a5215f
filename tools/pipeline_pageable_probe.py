"""bitrev_host_pipeline on pageable numpy arrays vs pinned tensors
(measurement tool): 8 arrays of 2^26 complex128 (1 GiB), out of place."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402

b, k = 26, 8
srcs = [np.full(1 << b, 1 + 2j, dtype=np.complex128) for _ in range(3)]
dsts = [np.empty_like(s) for s in srcs]
out = {}
for name, (S, D) in {"numpy": (srcs, dsts),
                     "pinned": ([torch.from_numpy(s).pin_memory() for s in srcs],
                                [torch.from_numpy(d).pin_memory() for d in dsts])}.items():
    seq_s = [S[i % 3] for i in range(k)]
    seq_d = [D[i % 3] for i in range(k)]
    br.bitrev_host_pipeline(seq_s[:2], b, seq_d[:2])
    t0 = time.perf_counter()
    br.bitrev_host_pipeline(seq_s, b, seq_d)
    out[name + "_gbs"] = 2 * k * srcs[0].nbytes / (time.perf_counter() - t0) / 1e9
print(json.dumps(out))
