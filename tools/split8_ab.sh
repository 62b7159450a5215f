#!/bin/bash
# 8-byte elements out of place as split 16-byte pairs (path 7,
# bitrev_oop_split8_kernel) against the rectangular default (path 3):
# parity of path 7 against the oracle (single arrays b = 13..24, batched rows,
# strided batches), then cfg3-8, cfg4 and b = 24 / 26 / 28 single arrays,
# interleaved rounds.
# Historical record: path 7 (bitrev_oop_split8_kernel and its launcher) was
# removed after this A/B: parity-green, 10 % slower (profiles/r02_split8_*).
O=gpurun_out
python - <<'PY' > $O/split8_parity.txt 2>&1
import torch
from paper_1708_01873_b200 import _core, _lib, oracle_permute
_lib.set_tile_path(8, False, 7)
bad = 0
for b in list(range(13, 25)) + [26]:
    for dt in (torch.float64, torch.complex64, torch.int64):
        x = torch.empty((1 << b) * 8, dtype=torch.uint8, device="cuda").random_(0, 256).view(dt)
        y = torch.empty_like(x)
        _core.launch_oop(x, y, b)
        ok = torch.equal(y.view(torch.uint8), oracle_permute(x, b).view(torch.uint8))
        bad += not ok
        print(b, dt, _lib.last_tile(), ok)
for b, rows in ((13, 64), (16, 256), (20, 8)):
    x = torch.empty((rows, 1 << b), dtype=torch.float64, device="cuda").normal_()
    y = torch.empty_like(x)
    _core.launch_oop(x, y, b)
    ok = all(torch.equal(y[r], oracle_permute(x[r], b)) for r in range(rows))
    bad += not ok
    print("batch", b, rows, _lib.last_tile(), ok)
    # strided rows inside a wider buffer
    big = torch.empty((rows, (1 << b) + 64), dtype=torch.float64, device="cuda").normal_()
    out = torch.zeros((rows, (1 << b) + 32), dtype=torch.float64, device="cuda")
    xs, ys = big[:, :1 << b], out[:, :1 << b]
    _core.launch_oop(xs, ys, b)
    ok = all(torch.equal(ys[r], oracle_permute(xs[r], b)) for r in range(rows)) and \
        bool((out[:, 1 << b:] == 0).all())
    bad += not ok
    print("strided", b, rows, _lib.last_tile(), ok)
print("BAD", bad)
PY
tail -1 $O/split8_parity.txt
: > $O/split8_ab.jsonl
for r in 1 2 3; do
  for p in 3 7; do
    for w in cfg3-8 cfg4; do
      python bench.py --workload $w --steps 20 --no-cpu-baseline --no-e2e --no-soak --tile-path $p 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'w': '$w', 'path': $p, 'value': d['value'], 'used': [d['config']['tile_bits'], d['config']['tile_path']], 'median_ms': d['step_ms']['median'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/split8_ab.jsonl
    done
  done
done
