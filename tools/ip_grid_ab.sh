# in-place pair kernel: persistent grid vs oversubscribed grids (cfg2), interleaved
O=gpurun_out
: > $O/ip_grid_ab.jsonl
for r in 1 2 3; do
  for m in 1 2 4 8; do
    BITREV_B200_IP_GRID_MULT=$m python bench.py --workload cfg2 --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'mult': $m, 'value': d['value'], 'median_ms': d['step_ms']['median']}))" >> $O/ip_grid_ab.jsonl
  done
done
