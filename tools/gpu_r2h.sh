# Round-2 batch: radix-8 against radix-4 drain at 7 stages (variants/lib_r4.so), cfg4-fft7 line.
set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x > $O/pytest_fft_r8.log 2>&1; echo pytest=$?; tail -1 $O/pytest_fft_r8.log
BITREV_B200_FFT_QZ=5 timeout 600 python -m pytest tests/test_gpu_fft_prepass.py -m gpu -q -x >> $O/pytest_fft_r8.log 2>&1; echo pytest_qz5=$?; tail -1 $O/pytest_fft_r8.log
: > $O/fft_r8_ab.txt
for r in 1 2 3; do
  for qz in 4 5; do
    BITREV_B200_FFT_QZ=$qz python tools/fft_stage_sweep.py 2>&1 | grep "stages=7" >> $O/fft_r8_ab.txt
    BITREV_B200_LIB=variants/lib_r4.so BITREV_B200_FFT_QZ=$qz python tools/fft_stage_sweep.py 2>&1 | grep "stages=7" | sed 's/^/R4 /' >> $O/fft_r8_ab.txt
  done
done
timeout 300 python bench.py --workload cfg4-fft7 --no-cpu-baseline > $O/bench_fft7.json 2>&1; echo bench=$?
