"""Host numpy arrays through the drop-in API (measurement tool): the
reference-style blocking calls on pageable numpy memory vs pinned torch host
tensors, 2^26 complex128 (1 GiB) out of place and in place."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402

b = 26
n = 1 << b
src = np.empty(n, dtype=np.complex128)
src.view(np.uint8)[:] = 7
dst = np.empty_like(src)
cfg = br.CobraConfig(6)
out = {}


def t(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 2 * src.nbytes / min(ts) / 1e9


out["numpy_oop_gbs"] = t(lambda: br.cobra_out_of_place(src, dst, cfg, b))
out["numpy_inplace_gbs"] = t(lambda: br.cobra_in_place(src, cfg, b))
ps = torch.from_numpy(src).pin_memory()
pd = torch.empty_like(ps).pin_memory()
out["pinned_oop_gbs"] = t(lambda: br.cobra_out_of_place(ps, pd, cfg, b))
out["pinned_inplace_gbs"] = t(lambda: br.cobra_in_place(ps, cfg, b))
print(json.dumps(out))
