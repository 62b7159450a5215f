#!/bin/bash
# 256-element-row FFT tiles (QX = 8) at 512 threads per CTA
# (variants/lib_fftnt512.so, built with -DBITREV_FFT_WIDE_NT=512: 16 warps
# share the drain, 32 load registers per thread) against 256 threads (the
# default build), both forced with BITREV_B200_FFT_QX=8, and the 128-element
# rows (BITREV_B200_FFT_QX=7); stage sweep, interleaved rounds.
# Historical record: the BITREV_FFT_WIDE_NT knob (Rect's thread-count
# parameter) was removed after this A/B (profiles/r02_fft_wide_nt_ab.txt:
# 512 threads tie at 1-5 stages, lose 4 % / 10 % at 6 / 7).
O=gpurun_out
BITREV_B200_LIB=variants/lib_fftnt512.so BITREV_B200_FFT_QX=8 timeout 900 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_nt512.log 2>&1; echo pytest=$?; tail -1 $O/pytest_fft_nt512.log
: > $O/fft_wide_nt_ab.txt
for r in 1 2 3; do
  echo "== nt512 round $r" >> $O/fft_wide_nt_ab.txt
  BITREV_B200_LIB=variants/lib_fftnt512.so BITREV_B200_FFT_QX=8 python tools/fft_stage_sweep.py >> $O/fft_wide_nt_ab.txt 2>&1
  echo "== nt256 round $r" >> $O/fft_wide_nt_ab.txt
  BITREV_B200_FFT_QX=8 python tools/fft_stage_sweep.py >> $O/fft_wide_nt_ab.txt 2>&1
  echo "== qx7 round $r" >> $O/fft_wide_nt_ab.txt
  BITREV_B200_FFT_QX=7 python tools/fft_stage_sweep.py >> $O/fft_wide_nt_ab.txt 2>&1
done
