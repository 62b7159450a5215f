"""Exercise every kernel path once at small sizes (for compute-sanitizer):
tile paths 0-6 for both families and all widths, short-row kernels (many
rows per CTA; in place also 64 KB rows), small/gather/swap fallbacks,
transpose, even-odd, explicit pairs, FFT pre-pass (tiles, short rows,
complete FFT of 64 KB rows), sharded unpack, host pipeline.  Each result is
checked against the torch oracle."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1708_01873_b200 as br  # noqa: E402
from paper_1708_01873_b200 import sharded  # noqa: E402

dev = torch.device("cuda", 0)
DT = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64, 16: torch.complex128}


def rnd(n, E, batch=None):
    shape = (n,) if batch is None else (batch, n)
    t = torch.empty(int(np.prod(shape)) * E, dtype=torch.uint8, device=dev).random_(0, 256)
    return t.view(DT[E]).view(shape)


def same(a, b):
    assert torch.equal(a.contiguous().view(torch.uint8), b.contiguous().view(torch.uint8))


checks = 0
saved = {(E, ip): (br.get_tile_bits(E, ip), br.get_tile_path(E, ip))
         for E in (4, 8, 16) for ip in (False, True)}
for E in (4, 8, 16):
    for path in (0, 1, 2, 3, 4, 5, 6):
        for b in (13, 14):
            for q in {4: (5, 6, 7), 8: (4, 5, 6, 7), 16: (3, 4, 5, 6)}[E]:
                for ip in (False, True):
                    if (path == 3 and ip) or (path >= 4 and not ip):
                        continue
                    br.set_tile_bits(E, ip, q)
                    br.set_tile_path(E, ip, path)
                    x = rnd(1 << b, E, batch=2)
                    ref = torch.stack([br.oracle_permute(r, b) for r in x])
                    if ip:
                        br.bitrev_batched_inplace(x, b)
                        same(x, ref)
                    else:
                        same(br.bitrev_batched(x, b), ref)
                    checks += 1
        for ip in (False, True):
            br.set_tile_bits(E, ip, saved[(E, ip)][0])
            br.set_tile_path(E, ip, saved[(E, ip)][1])
for E in (1, 2, 4, 8, 16):  # small path, and element-wise fallbacks via misalignment
    x = rnd((1 << 10) + 1, E)
    v = x[1:]
    same(br.bitrev_batched(v.view(1, -1), 10), br.oracle_permute(v, 10).view(1, -1))
    y = rnd((1 << 15) + 1, E)[1:]
    ref = br.oracle_permute(y, 15)
    out = torch.empty_like(y)
    br.cobra_out_of_place(y, out, br.CobraConfig(0), 15)
    same(out, ref)
    br.cobra_in_place(y, br.CobraConfig(0), 15)
    same(y, ref)
    checks += 3
for E in (4, 8, 16):  # short-row kernel: many rows per CTA, padded rows
    for b, batch in ((5, 333), (9, 17)):
        for pad in (0, 16):
            buf = rnd(((1 << b) + pad) * batch, E).view(batch, -1)
            rows = buf[:, :1 << b]
            ref = torch.stack([br.oracle_permute(r.contiguous(), b) for r in rows])
            same(br.bitrev_batched(rows, b), ref)
            br.bitrev_batched_inplace(rows, b)
            same(rows, ref)
            checks += 2
x = rnd(1 << 13, 8, batch=1024)  # in place: 64 KB rows in a 64 MiB batch
ref = torch.stack([br.oracle_permute(r, 13) for r in x])
br.bitrev_batched_inplace(x, 13)
same(x, ref)
checks += 1
t = rnd(1 << 12, 8)
w = t.clone()
br.transpose_square_inplace(w, 6)
same(w, t.view(64, 64).t().reshape(-1))
w = t.clone()
br.even_odd_permute(w, 12)
same(w, torch.cat([t[0::2], t[1::2]]))
r = br.rev_index_array(12).cpu().numpy()
i = np.arange(1 << 12)
a = t.clone()
br.apply_schedule(a, br.SwapSchedule(12, np.stack([i[i < r], r[i < r]], 1)))
same(a, br.oracle_permute(t, 12))
z = torch.randn(1 << 14, dtype=torch.complex64, device=dev)
for stages in (0, 3, 7):
    br.bitrev_dit_prepass(z, 14, stages)
br.bitrev_dit_prepass(z[:1 << 10], 10, 10)
zz = torch.randn(6, 1 << 13, dtype=torch.complex64, device=dev)
br.bitrev_dit_prepass(zz, 13, 13)  # complete FFT of 64 KB rows
br.bitrev_dit_prepass(zz.view(-1)[:5 << 10].view(5, 1 << 10), 10, 6)  # short rows, batched
g = rnd(1 << 16, 8)
same(torch.cat(sharded.emulate_sharded(g, 16, 4, 2)), br.oracle_permute(g, 16))
hosts = [torch.randn(1 << 14, dtype=torch.float64).pin_memory() for _ in range(3)]
refs = [br.oracle_permute(h, 14) for h in hosts]
br.bitrev_host_pipeline(hosts, 14)
for h, rf in zip(hosts, refs):
    same(h, rf)
torch.cuda.synchronize()
print(f"sanitize_paths ok: {checks} tile/fallback checks + aux paths")
