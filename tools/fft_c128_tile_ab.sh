#!/bin/bash
# complex128, 1-5 stages: square Q6 tiles with shuffle butterflies
# (bitrev_fft_tile16_kernel, default) against the rectangular (6,4) tiles with
# the radix-4 drain (BITREV_B200_FFT_C128_TILE=0); FFT parity tests first,
# then the complex128 stage sweep (2048 rows of 2^16), interleaved rounds.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_c128tile.log 2>&1; echo pytest=$?; tail -1 $O/pytest_c128tile.log
: > $O/fft_c128_tile_ab.txt
for r in 1 2 3; do
  for v in 1 0; do
    echo "== tile $v round $r" >> $O/fft_c128_tile_ab.txt
    BITREV_B200_FFT_C128_TILE=$v python tools/fft_stage_sweep.py --c128 >> $O/fft_c128_tile_ab.txt 2>&1
  done
done
