# cfg1 (2^20 complex128): the Q5 tier's tile kernel at 1 / 3 / 4 CTAs/SM (BITREV_B200_SMALL_MINB), flushed and L2-hot.
O=gpurun_out
: > $O/cfg1_minb_ab.jsonl
for r in 1 2 3; do
 for m in 1 3 4; do
  BITREV_B200_SMALL_MINB=$m python bench.py --workload cfg1 --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'minb': $m, 'value': d['value'], 'median_ms': d['step_ms']['median'], 'l2hot': d['l2_hot']['value'], 'copy': d['roofline']['torch_copy_same_harness_gbs']}))" >> $O/cfg1_minb_ab.jsonl
 done
done
