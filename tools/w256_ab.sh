# 32-byte stores (STG.256) in the rectangular out-of-place tiles: parity + A/B
# Historical record: the knob this A/B switched was removed from the library after
# the measurement (result under profiles/r02_*); rerunning measures the default twice.
O=gpurun_out
BITREV_B200_W256=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py -m gpu -q -x -k "oop or out_of_place or cfg3 or cfg4 or every_element" > $O/pytest_w256.log 2>&1; echo pytest=$?; tail -1 $O/pytest_w256.log
: > $O/w256_ab.jsonl
for r in 1 2 3; do
  for w in 0 1; do
    for wl in cfg3-8 cfg4 cfg3-4; do
      BITREV_B200_W256=$w python bench.py --workload $wl --steps 20 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'w256': $w, 'w': '$wl', 'value': d['value'], 'median_ms': d['step_ms']['median']}))" >> $O/w256_ab.jsonl
    done
  done
done
