#!/bin/bash
# 1-3 fused stages: the 256-element-row tiles through the radix-8 drain
# (BITREV_B200_FFT_QX=8) against the default 128-element rows (radix-4
# drain), stage sweep, interleaved rounds; parity under the knob first.
O=gpurun_out
BITREV_B200_FFT_QX=8 timeout 900 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_qx8_low.log 2>&1; echo pytest=$?; tail -1 $O/pytest_fft_qx8_low.log
: > $O/fft_qx8_low_ab.txt
for r in 1 2 3; do
  for q in 7 8; do
    echo "== qx $q round $r" >> $O/fft_qx8_low_ab.txt
    BITREV_B200_FFT_QX=$q python tools/fft_stage_sweep.py >> $O/fft_qx8_low_ab.txt 2>&1
  done
done
