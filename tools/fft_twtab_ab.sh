#!/bin/bash
# Radix-8 drain twiddles: the W_4 / W_8 multiples of stages 5-7 read from the
# per-CTA table (variants/lib_twtab.so, -DBITREV_FFT_TW_TABLE=1) or of stage 7
# only (variants/lib_twtab2.so, =2) instead of formed per pass (default).
# Parity under each variant, then the stage sweep and cfg4-fft7, interleaved.
# Historical record: the BITREV_FFT_TW_TABLE knob was removed after this A/B
# (profiles/r02_fft_twtab_ab.*: 7 stages -6 / -16 % from register spills).
O=gpurun_out
for v in twtab twtab2; do
  BITREV_B200_LIB=variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_$v.log 2>&1; echo $v pytest=$?; tail -1 $O/pytest_$v.log
done
: > $O/fft_twtab_ab.txt
: > $O/fft_twtab_ab.jsonl
for r in 1 2 3; do
  for v in default twtab twtab2; do
    if [ $v = default ]; then unset BITREV_B200_LIB; else export BITREV_B200_LIB=variants/lib_$v.so; fi
    echo "== $v round $r" >> $O/fft_twtab_ab.txt
    python tools/fft_stage_sweep.py >> $O/fft_twtab_ab.txt 2>&1
    python bench.py --workload cfg4-fft7 --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'lib': '$v', 'value': d['value'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/fft_twtab_ab.jsonl
  done
done
unset BITREV_B200_LIB
