#!/bin/bash
# float64 / complex64 out of place: rectangular tiles with 2 KB destination
# rows (QX = 8, QZ = 5: 64 KB tiles, the byte geometry of the float32
# default) against the default 1 KB rows (QX = 7, QZ = 5: 32 KB tiles),
# parity of the new shape, then cfg3-8 and cfg4, interleaved rounds.
O=gpurun_out
python - <<'PY' > $O/rect_e8_q8_parity.txt 2>&1
import torch
from paper_1708_01873_b200 import _core, _lib, oracle_permute
_lib.set_tile_bits(8, False, 8); _lib.set_tile_path(8, False, 3)
bad = 0
for b in (13, 14, 16, 20, 24, 26):
    x = torch.empty((1 << b) * 8, dtype=torch.uint8, device="cuda").random_(0, 256).view(torch.float64)
    y = torch.empty_like(x)
    _core.launch_oop(x, y, b)
    ok = torch.equal(y.view(torch.uint8), oracle_permute(x, b).view(torch.uint8))
    bad += not ok
    print(b, _lib.last_tile(), ok)
x = torch.empty((64, 1 << 16), dtype=torch.complex64, device="cuda").normal_()
y = torch.empty_like(x)
_core.launch_oop(x, y, 16)
ok = all(torch.equal(y[r], oracle_permute(x[r], 16)) for r in range(64))
bad += not ok
print("batch", _lib.last_tile(), ok)
print("BAD", bad)
PY
tail -1 $O/rect_e8_q8_parity.txt
: > $O/rect_e8_q8_ab.jsonl
for r in 1 2 3; do
  for q in 7 8; do
    for w in cfg3-8 cfg4; do
      python bench.py --workload $w --steps 20 --no-cpu-baseline --no-e2e --no-soak --tile-bits $q --tile-path 3 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'w': '$w', 'qx': $q, 'value': d['value'], 'used': [d['config']['tile_bits'], d['config']['tile_path']], 'median_ms': d['step_ms']['median']}))" >> $O/rect_e8_q8_ab.jsonl
    done
  done
done
