#!/bin/bash
# cfg3-8 (2^30 float64 out of place): square Q7 register tiles at 512 threads
# (1 KB runs on both sides, path 0) against the default rectangular tiles
# (1 KB destination rows, 256-byte source pieces, path 3), interleaved rounds.
O=gpurun_out
: > $O/oop_e8_q7_ab.jsonl
for r in 1 2 3; do
  for tp in "7 3" "7 0"; do
    set -- $tp
    python bench.py --workload cfg3-8 --steps 10 --no-cpu-baseline --no-e2e --no-soak --tile-bits $1 --tile-path $2 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'q': $1, 'path': $2, 'value': d['value'], 'used': [d['config']['tile_bits'], d['config']['tile_path']], 'median_ms': d['step_ms']['median']}))" >> $O/oop_e8_q7_ab.jsonl
  done
done
