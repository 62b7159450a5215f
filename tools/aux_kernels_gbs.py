"""GB/s of the auxiliary entry points at cfg2's size (measurement tool):
transpose_square_inplace at h = 13 (8192 x 8192 float64, 512 MiB) and
even_odd_permute at b = 26 float64, beside a torch copy_ of the same bytes.
even_odd moves its 512 MiB twice (two in-place reversals): GB/s are reported
on the entry point's 2*n*E bytes."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    ts.sort()
    return ts[len(ts) // 2]


x = torch.empty(1 << 26, dtype=torch.float64, device="cuda").normal_()
y = torch.empty_like(x)
nb = 2 * x.numel() * 8
out = {"bytes_per_call": nb,
       "transpose_h13_gbs": nb / t(lambda: br.transpose_square_inplace(x, 13)) / 1e9,
       "even_odd_b26_gbs": nb / t(lambda: br.even_odd_permute(x, 26)) / 1e9,
       "bitrev_inplace_b26_gbs": nb / t(lambda: br.cobra_in_place(x, br.CobraConfig(6), 26)) / 1e9,
       "torch_copy_gbs": nb / t(lambda: y.copy_(x)) / 1e9}
print(json.dumps(out))
