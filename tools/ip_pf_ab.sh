#!/bin/bash
# In-place pairs with an L2 bulk-prefetch lookahead (BITREV_IP_PF = 1 / 2
# items ahead of the register loads; variants/lib_ippf{1,2}.so built with
# python -m paper_1708_01873_b200.build --out variants/lib_ippfN.so -DBITREV_IP_PF=N)
# against the default library: in-place parity on the variant, then cfg2
# (2^26 float64 in place), interleaved rounds.
# Historical record: the BITREV_IP_PF knob (a second pair cursor issuing
# cp.async.bulk.prefetch.L2 per tile row) was removed after this A/B:
# profiles/r02_ip_pf_ab.jsonl, 8-10 % slower.
O=gpurun_out
BITREV_B200_LIB=variants/lib_ippf1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -x -k "inplace or in_place" > $O/pytest_ippf.log 2>&1; echo pytest=$?; tail -1 $O/pytest_ippf.log
: > $O/ip_pf_ab.jsonl
for r in 1 2 3; do
  for v in default ippf1 ippf2; do
    if [ $v = default ]; then unset BITREV_B200_LIB; else export BITREV_B200_LIB=variants/lib_$v.so; fi
    python bench.py --workload cfg2 --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'lib': '$v', 'value': d['value'], 'median_ms': d['step_ms']['median'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/ip_pf_ab.jsonl
  done
done
unset BITREV_B200_LIB
