#!/bin/bash
# Rectangular tiles flipped: long (1 KB) source pieces, short destination rows
# (QZ > QX) against the default (1 KB destination rows, 256-byte pieces).
# cfg3-8 and cfg3-4, interleaved rounds.  Result: profiles/r02_rect_flip_ab.jsonl.
# The flipped instantiations RECT(8,5,7) RECT(8,6,7) RECT(4,6,7) were removed
# from dispatch_oop_rect after this A/B; add them back to rerun it.
O=gpurun_out
: > $O/rect_flip_ab.jsonl
run() {  # workload q qz
  BITREV_B200_RECT_QZ=$3 python bench.py --workload $1 --steps 10 --no-cpu-baseline --no-e2e --no-soak --tile-bits $2 --tile-path 3 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'w': '$1', 'qx': $2, 'qz': $3, 'value': d['value'], 'used': [d['config']['tile_bits'], d['config']['tile_path']]}))" >> $O/rect_flip_ab.jsonl
}
for r in 1 2; do
  run cfg3-8 7 5; run cfg3-8 5 7; run cfg3-8 6 7
  run cfg3-4 8 6; run cfg3-4 6 7
done
# parity of the flipped shapes (b = 22, every element against the oracle)
for cfg in "8 5 7" "8 6 7" "4 6 7"; do
  set -- $cfg
  BITREV_B200_RECT_QZ=$3 python - $1 $2 <<'PY' >> $O/rect_flip_ab.jsonl
import sys, json, torch
from paper_1708_01873_b200 import _core, _lib, oracle_permute
E, q = int(sys.argv[1]), int(sys.argv[2])
dt = {4: torch.float32, 8: torch.float64}[E]
b = 22
x = torch.empty((1 << b) * E, dtype=torch.uint8, device="cuda").random_(0, 256).view(dt)
y = torch.empty_like(x)
_lib.set_tile_bits(E, False, q); _lib.set_tile_path(E, False, 3)
_core.launch_oop(x, y, b)
torch.cuda.synchronize()
ok = torch.equal(y.view(torch.uint8), oracle_permute(x, b).view(torch.uint8))
print(json.dumps({"parity": ok, "E": E, "qx": q, "used": list(_lib.last_tile())}))
PY
done
