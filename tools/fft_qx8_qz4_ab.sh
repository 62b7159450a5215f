#!/bin/bash
# 256-element-row FFT tiles with 128-byte source pieces (QX = 8, QZ = 4: 32 KB
# tiles, 2 CTAs/SM; BITREV_B200_FFT_QX=8 BITREV_B200_FFT_QZ=4) against QX = 8
# QZ = 5 (64 KB, 1 CTA/SM) and QX = 7 QZ = 5; parity under the new shape,
# stage sweep, interleaved rounds.
# Historical record: the (8, 8, 4, S) instantiations were removed after this
# A/B (profiles/r02_fft_qx8_qz4_ab.txt: 3-21 % below QZ = 5 at 1-7 stages).
O=gpurun_out
BITREV_B200_FFT_QX=8 BITREV_B200_FFT_QZ=4 timeout 900 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_qz4w.log 2>&1; echo pytest=$?; tail -1 $O/pytest_fft_qz4w.log
: > $O/fft_qx8_qz4_ab.txt
for r in 1 2 3; do
  echo "== q8z4 round $r" >> $O/fft_qx8_qz4_ab.txt
  BITREV_B200_FFT_QX=8 BITREV_B200_FFT_QZ=4 python tools/fft_stage_sweep.py >> $O/fft_qx8_qz4_ab.txt 2>&1
  echo "== q8z5 round $r" >> $O/fft_qx8_qz4_ab.txt
  BITREV_B200_FFT_QX=8 python tools/fft_stage_sweep.py >> $O/fft_qx8_qz4_ab.txt 2>&1
  echo "== q7z5 round $r" >> $O/fft_qx8_qz4_ab.txt
  BITREV_B200_FFT_QX=7 BITREV_B200_FFT_QZ=5 python tools/fft_stage_sweep.py >> $O/fft_qx8_qz4_ab.txt 2>&1
done
