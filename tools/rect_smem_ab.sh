# out-of-place rectangular tiles: occupancy A/B through padded shared memory
O=gpurun_out
: > $O/rect_smem_ab.jsonl
for r in 1 2 3; do
  for kb in 0 120; do
    for w in cfg3-8 cfg4; do
      BITREV_B200_RECT_SMEM_KB=$kb python bench.py --workload $w --steps 20 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'smem_kb': $kb, 'w': '$w', 'value': d['value'], 'median_ms': d['step_ms']['median']}))" >> $O/rect_smem_ab.jsonl
    done
  done
done
