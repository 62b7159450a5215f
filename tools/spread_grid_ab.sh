#!/bin/bash
# ~5 tiles per CTA against persistent grids for the sharded pack / fused
# scatter (BITREV_B200_PACK_TILES_PER_CTA) and the FFT pre-pass tiles
# (BITREV_B200_FFT_TILES_PER_CTA): cfg5's local phases, the complex64 /
# complex128 stage sweeps and the cfg4-fft7 line, interleaved; parity under
# the spread grids first.
O=gpurun_out
BITREV_B200_PACK_TILES_PER_CTA=5 BITREV_B200_FFT_TILES_PER_CTA=5 timeout 900 python -m pytest tests/test_gpu_fft_prepass.py tests/test_gpu_baseline_sizes.py tests/test_gpu_sharded_e2e.py -m gpu -q -x -k "fft or prepass or cfg5 or pack or unpack or sharded or wide or strided" > $O/pytest_spread.log 2>&1; echo pytest=$?; tail -1 $O/pytest_spread.log
: > $O/spread_grid_ab.txt
: > $O/spread_grid_ab.jsonl
for r in 1 2; do
  for t in 5 0; do
    export BITREV_B200_PACK_TILES_PER_CTA=$t BITREV_B200_FFT_TILES_PER_CTA=$t
    echo "== tpc $t round $r" >> $O/spread_grid_ab.txt
    python tools/fft_stage_sweep.py >> $O/spread_grid_ab.txt 2>&1
    python tools/fft_stage_sweep.py --c128 >> $O/spread_grid_ab.txt 2>&1
    python tools/cfg5_phases.py | sed "s/^{/{\"tpc\": $t, /" >> $O/spread_grid_ab.jsonl
    python bench.py --workload cfg4-fft7 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'tpc': $t, 'w': 'cfg4-fft7', 'value': d['value'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/spread_grid_ab.jsonl
  done
done
unset BITREV_B200_PACK_TILES_PER_CTA BITREV_B200_FFT_TILES_PER_CTA
