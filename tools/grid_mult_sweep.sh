#!/bin/bash
# Persistent tile kernels launched with M x the resident CTAs: the resident
# CTAs start on tiles M * (resident grid) apart instead of adjacent ones.
# Out of place (BITREV_B200_OOP_GRID_MULT) over cfg3-16 / cfg3-8 / cfg3-4 /
# cfg4 / cfg5 (N = 1), in place (BITREV_B200_IP_GRID_MULT) over cfg2.
O=gpurun_out
: > $O/grid_mult_sweep.jsonl
run() {  # env mult workload
  env $1=$2 python bench.py --workload $3 --steps 10 --no-cpu-baseline --no-e2e --no-soak --no-sweep 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'knob': '$1', 'mult': $2, 'w': '$3', 'value': d['value']}))" >> $O/grid_mult_sweep.jsonl
}
for r in 1 2; do
  for m in 1 32 128 256 512; do
    for w in cfg3-16 cfg3-8 cfg5; do run BITREV_B200_OOP_GRID_MULT $m $w; done
  done
  for m in 1 8 16 32 64; do
    for w in cfg4 cfg3-4; do run BITREV_B200_OOP_GRID_MULT $m $w; done
  done
  for m in 1 16 64 256; do run BITREV_B200_IP_GRID_MULT $m cfg2; done
done
