#!/bin/bash
# complex128 square-tile shuffle stages, select-free form (each lane scales
# its own value, swaps, adds with a per-lane sign): tile path for 1-5 stages
# (BITREV_B200_FFT_C128_TILE_MAX=5) against the rectangular radix-4 drain
# (BITREV_B200_FFT_C128_TILE=0); parity over 1-5 stages first.
O=gpurun_out
BITREV_B200_FFT_C128_TILE_MAX=5 timeout 900 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_c128tile2.log 2>&1; echo pytest=$?; tail -1 $O/pytest_c128tile2.log
: > $O/fft_c128_tile2_ab.txt
for r in 1 2 3; do
  echo "== tile round $r" >> $O/fft_c128_tile2_ab.txt
  BITREV_B200_FFT_C128_TILE_MAX=5 python tools/fft_stage_sweep.py --c128 >> $O/fft_c128_tile2_ab.txt 2>&1
  echo "== rect round $r" >> $O/fft_c128_tile2_ab.txt
  BITREV_B200_FFT_C128_TILE=0 python tools/fft_stage_sweep.py --c128 >> $O/fft_c128_tile2_ab.txt 2>&1
done
