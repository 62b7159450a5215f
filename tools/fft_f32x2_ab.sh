#!/bin/bash
# complex64 FFT pre-pass math on the packed FP32 pipe (FADD2/FMUL2/FFMA2,
# default) against scalar FADD/FMUL/FFMA (variants/lib_nof32x2.so, built with
# python -m paper_1708_01873_b200.build --out variants/lib_nof32x2.so
# -DBITREV_FFT_F32X2=0): FFT parity tests on the default library, then the
# stage sweep (20 back-to-back launches, cfg4 shape) and the cfg4-fft7 bench
# line, interleaved rounds.
# Historical record: the packed path (cadd/csub/cmul float2 specialisations on
# add/sub/mul/fma.rn.f32x2, BITREV_FFT_F32X2) was removed after this A/B
# (profiles/r02_fft_f32x2_ab.*: 7 stages 5-8 % slower, 1-6 stages within 1 %).
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fft_prepass.py tests/test_gpu_plan.py -m gpu -q -x > $O/pytest_f32x2.log 2>&1; echo pytest=$?; tail -1 $O/pytest_f32x2.log
: > $O/fft_f32x2_ab.txt
: > $O/fft_f32x2_ab.jsonl
for r in 1 2 3; do
  for v in default nof32x2; do
    if [ $v = default ]; then unset BITREV_B200_LIB; else export BITREV_B200_LIB=variants/lib_nof32x2.so; fi
    echo "== $v round $r" >> $O/fft_f32x2_ab.txt
    python tools/fft_stage_sweep.py >> $O/fft_f32x2_ab.txt 2>&1
    python bench.py --workload cfg4-fft7 --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'lib': '$v', 'value': d['value'], 'median_ms': d['step_ms']['median'], 'clocks': d['clocks']['sm_mhz']}))" >> $O/fft_f32x2_ab.jsonl
  done
done
unset BITREV_B200_LIB
