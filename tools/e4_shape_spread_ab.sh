#!/bin/bash
# float32 out of place (cfg3-4): the default rect (8,6) 64 KB tiles (1 CTA/SM,
# persistent) against 32 KB shapes that run 2 CTAs/SM -- rect (7,6) and rect
# (8,5) -- each with persistent and ~5-tiles-per-CTA grids.
# Historical record: RECT(4, 8, 5) was instantiated for this A/B only and
# removed (profiles/r02_e4_shape_spread_ab.jsonl: the default stays best).
O=gpurun_out
: > $O/e4_shape_spread_ab.jsonl
run() {  # label q qz tpc
  env ${3:+BITREV_B200_RECT_QZ=$3} BITREV_B200_OOP_TILES_PER_CTA=$4 python bench.py --workload cfg3-4 --steps 10 --no-cpu-baseline --no-e2e --no-soak --no-sweep --tile-bits $2 --tile-path 3 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'shape': '$1', 'tpc': $4, 'value': d['value'], 'used': [d['config']['tile_bits'], d['config']['tile_path']]}))" >> $O/e4_shape_spread_ab.jsonl
}
for r in 1 2; do
  for t in 0 5; do
    run "8,6" 8 "" $t
    run "7,6" 7 "" $t
    run "8,5" 8 5 $t
  done
done
