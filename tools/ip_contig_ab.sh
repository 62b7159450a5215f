#!/bin/bash
# In-place pairs: each CTA takes K consecutive pairs of the compact enumeration
# (BITREV_B200_IP_CONTIG=K, grid = pairs / K) instead of every grid-th pair of
# a persistent grid (0); cfg2 and b = 28 float64 in place, interleaved; parity
# under K = 4 first.
# Historical record: the BITREV_B200_IP_CONTIG knob (TileArgs.per_cta) was
# removed after this A/B (profiles/r02_ip_contig_ab.jsonl: every K slower).
O=gpurun_out
BITREV_B200_IP_CONTIG=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_baseline_sizes.py -m gpu -q -x -k "inplace or in_place or cfg2" > $O/pytest_ipcontig.log 2>&1; echo pytest=$?; tail -1 $O/pytest_ipcontig.log
: > $O/ip_contig_ab.jsonl
for r in 1 2; do
  for k in 0 1 2 4 8 16 56; do
    BITREV_B200_IP_CONTIG=$k python bench.py --workload cfg2 --steps 20 --no-cpu-baseline --no-e2e --no-soak 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'k': $k, 'w': 'cfg2', 'value': d['value']}))" >> $O/ip_contig_ab.jsonl
  done
done
