# in-place E=8 pair kernel: 256 threads x 1 CTA/SM vs 128 threads x 2 CTAs/SM
# Historical record: the knob this A/B switched was removed from the library after
# the measurement (result under profiles/r02_*); rerunning measures the default twice.
O=gpurun_out
BITREV_B200_IP_NT=128 timeout 600 python -m pytest tests/test_gpu_baseline_sizes.py -m gpu -q -x -k "cfg2" > $O/pytest_ipnt.log 2>&1; echo pytest=$?; tail -1 $O/pytest_ipnt.log
: > $O/ip_nt_ab.jsonl
for r in 1 2 3; do
  for nt in 256 128; do
    BITREV_B200_IP_NT=$nt python bench.py --workload cfg2 --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'nt': $nt, 'value': d['value']}))" >> $O/ip_nt_ab.jsonl
  done
done
