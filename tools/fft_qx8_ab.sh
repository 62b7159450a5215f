#!/bin/bash
# complex64 FFT pre-pass with 256-element destination rows (QX = 8, two
# 128-element FFT blocks per row, radix-8 drain, 4..7 stages, 1 CTA/SM)
# against the default 128-element rows (QX = 7, 2 CTAs/SM):
# BITREV_B200_FFT_QX=8 selects the wide tiles.  Parity (the FFT test file
# under the knob), then the stage sweep and the cfg4-fft7 bench line,
# interleaved rounds.
O=gpurun_out
BITREV_B200_FFT_QX=8 timeout 900 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_qx8.log 2>&1; echo pytest=$?; tail -1 $O/pytest_fft_qx8.log
: > $O/fft_qx8_ab.txt
: > $O/fft_qx8_ab.jsonl
for r in 1 2 3; do
  for q in 7 8; do
    echo "== qx $q round $r" >> $O/fft_qx8_ab.txt
    BITREV_B200_FFT_QX=$q python tools/fft_stage_sweep.py >> $O/fft_qx8_ab.txt 2>&1
    BITREV_B200_FFT_QX=$q python bench.py --workload cfg4-fft7 --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'qx': $q, 'value': d['value'], 'median_ms': d['step_ms']['median'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/fft_qx8_ab.jsonl
  done
done
