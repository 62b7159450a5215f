#!/bin/bash
# complex64, 6-7 stages on 128-element rows: radix-16 drain (one layout
# exchange; variants/lib_r16.so, -DBITREV_FFT_R16=1) against the radix-8
# drain (two exchanges; default).  Parity under the variant, then the stage
# sweep and the cfg4-fft7 bench line, interleaved rounds.
# Historical record: the radix-16 drain (BITREV_FFT_R16) was removed after
# this A/B (profiles/r02_fft_r16_ab.*: parity-green, 7 stages -3 to -5 %,
# 6 stages a tie).
O=gpurun_out
BITREV_B200_LIB=variants/lib_r16.so timeout 900 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_r16.log 2>&1; echo pytest=$?; tail -1 $O/pytest_r16.log
: > $O/fft_r16_ab.txt
: > $O/fft_r16_ab.jsonl
for r in 1 2 3; do
  for v in default r16; do
    if [ $v = default ]; then unset BITREV_B200_LIB; else export BITREV_B200_LIB=variants/lib_r16.so; fi
    echo "== $v round $r" >> $O/fft_r16_ab.txt
    python tools/fft_stage_sweep.py >> $O/fft_r16_ab.txt 2>&1
    python bench.py --workload cfg4-fft7 --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'lib': '$v', 'value': d['value'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/fft_r16_ab.jsonl
  done
done
unset BITREV_B200_LIB
