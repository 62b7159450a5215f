# Round-2 batch: complex64 FFT with 128- vs 256-byte source pieces (BITREV_B200_FFT_QZ), parity and stage sweep.
set -u
O=gpurun_out
BITREV_B200_FFT_QZ=5 timeout 600 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_qz5.log 2>&1; echo pytest_qz5=$?; tail -2 $O/pytest_fft_qz5.log
: > $O/fft_qz_ab.txt
for r in 1 2 3; do
  python tools/fft_stage_sweep.py >> $O/fft_qz_ab.txt 2>&1
  BITREV_B200_FFT_QZ=5 python tools/fft_stage_sweep.py >> $O/fft_qz_ab.txt 2>&1
done
