# Round-2 batch: radix-8 drain from 4 stages on (variants/lib_r8from4.so) against the default.
set -u
O=gpurun_out
BITREV_B200_LIB=variants/lib_r8from4.so timeout 600 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_r8b.log 2>&1; echo pytest_r8from4=$?; tail -1 $O/pytest_fft_r8b.log
: > $O/fft_r8_from4_ab.txt
for r in 1 2 3; do
  python tools/fft_stage_sweep.py 2>&1 | grep "stages=[4567]" >> $O/fft_r8_from4_ab.txt
  BITREV_B200_LIB=variants/lib_r8from4.so python tools/fft_stage_sweep.py 2>&1 | grep "stages=[4567]" | sed 's/^/R8 /' >> $O/fft_r8_from4_ab.txt
done
