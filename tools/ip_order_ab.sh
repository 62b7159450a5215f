# in-place visit order A/B on cfg2 (interleaved rounds)
O=gpurun_out
: > $O/ip_order_ab.jsonl
for r in 1 2 3; do
  for o in 2 0 1 273 546; do
    BITREV_B200_ORDER_IP=$o python bench.py --workload cfg2 --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'order': $o, 'value': d['value'], 'median_ms': d['step_ms']['median']}))" >> $O/ip_order_ab.jsonl
  done
done
