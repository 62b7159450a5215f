#!/bin/bash
# Out-of-place tile kernels (square and rectangular, persistent with the next
# tile's loads in flight) launched with 1x / 2x / 4x / 16x the resident CTAs
# (BITREV_B200_OOP_GRID_MULT), cfg3-16 / cfg3-8 / cfg3-4 / cfg4, interleaved.
O=gpurun_out
: > $O/oop_grid_ab.jsonl
for r in 1 2; do
  for m in ${MULTS:-1 2 4 16}; do
    for w in cfg3-16 cfg3-8 cfg3-4 cfg4; do
      BITREV_B200_OOP_GRID_MULT=$m python bench.py --workload $w --steps 10 --no-cpu-baseline --no-e2e --no-soak --no-sweep 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'mult': $m, 'w': '$w', 'value': d['value']}))" >> $O/oop_grid_ab.jsonl
    done
  done
done
