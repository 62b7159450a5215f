# Round-2 batch: FFT stage-7 warp-shuffle variant (variants/lib_s7d.so) against the shared-memory exchange.
set -u
O=gpurun_out
BITREV_B200_FFT_QZ=5 timeout 600 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_s7.log 2>&1; echo pytest_qz5=$?; tail -1 $O/pytest_fft_s7.log
timeout 600 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x >> $O/pytest_fft_s7.log 2>&1; echo pytest_qz4=$?; tail -1 $O/pytest_fft_s7.log
: > $O/fft_s7_ab.txt
for r in 1 2 3; do
  python tools/fft_stage_sweep.py >> $O/fft_s7_ab.txt 2>&1
  BITREV_B200_FFT_QZ=5 python tools/fft_stage_sweep.py >> $O/fft_s7_ab.txt 2>&1
  BITREV_B200_LIB=variants/lib_s7d.so python tools/fft_stage_sweep.py | sed 's/^E=8/D E=8/' >> $O/fft_s7_ab.txt 2>&1
  BITREV_B200_LIB=variants/lib_s7d.so BITREV_B200_FFT_QZ=5 python tools/fft_stage_sweep.py | sed 's/^E=8/D E=8/' >> $O/fft_s7_ab.txt 2>&1
done
