#!/bin/bash
# Out-of-place grids at ~5 tiles per CTA (default) against persistent grids
# (BITREV_B200_OOP_TILES_PER_CTA=0): parity of the out-of-place tests under the
# new default, the bench workloads, and the float64 / complex128 size curve
# (b = 20..28, L2 flushed below 1 GiB), interleaved.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mid_sizes.py tests/test_gpu_golden.py -m gpu -q -x -k "oop or out_of_place or batched or mid or cobra" > $O/pytest_tpc.log 2>&1; echo pytest=$?; tail -1 $O/pytest_tpc.log
: > $O/oop_tpc_ab.jsonl
for r in 1 2; do
  for t in 5 0; do
    for w in cfg3-16 cfg3-8 cfg4 cfg5 cfg1; do
      BITREV_B200_OOP_TILES_PER_CTA=$t python bench.py --workload $w --steps 10 --no-cpu-baseline --no-e2e --no-soak --no-sweep 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'tpc': $t, 'w': '$w', 'value': d['value']}))" >> $O/oop_tpc_ab.jsonl
    done
    BITREV_B200_OOP_TILES_PER_CTA=$t python tools/size_curve.py --bits 20 21 22 23 24 25 26 27 28 --widths 8 16 --reps 20 2>/dev/null | \
      python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d.get('kind')=='cell' and not d['inplace']: print(json.dumps({'tpc': $t, 'E': d['E'], 'b': d['b'], 'gbs': d['gbs']}))" >> $O/oop_tpc_ab.jsonl
  done
done
