#!/bin/bash
# Rectangular out-of-place tiles with __launch_bounds__ min 2 CTAs/SM
# (variants/lib_rectminb2.so, -DBITREV_RECT_MINB=2: float32 (8,6) and the
# batched float64 (8,5) fall from 158 to 128 registers, 1 -> 2 CTAs/SM)
# against the default; cfg3-4, cfg4 and cfg3-8 (control), interleaved.
# Historical record: the BITREV_RECT_MINB knob was removed after this A/B
# (profiles/r02_rect_minb_ab.jsonl: float32 -7 %, batched float64 -5 % at 2
# CTAs/SM).  Its 'default' cfg3-8 rows (5365) are not the default kernel: an
# explicit minimum of 1 let ptxas give the (7,5) tiles 168 registers (1 CTA/SM)
# where the product's __launch_bounds__(256) settles at 122 (2 CTAs/SM).
O=gpurun_out
BITREV_B200_LIB=variants/lib_rectminb2.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mid_sizes.py -m gpu -q -x -k "oop or out_of_place or batched or mid" > $O/pytest_rectminb.log 2>&1; echo pytest=$?; tail -1 $O/pytest_rectminb.log
: > $O/rect_minb_ab.jsonl
for r in 1 2 3; do
  for v in default rectminb2; do
    if [ $v = default ]; then unset BITREV_B200_LIB; else export BITREV_B200_LIB=variants/lib_$v.so; fi
    for w in cfg3-4 cfg4 cfg3-8; do
      python bench.py --workload $w --steps 20 --no-cpu-baseline --no-e2e --no-soak 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'lib': '$v', 'w': '$w', 'value': d['value'], 'used': [d['config']['tile_bits'], d['config']['tile_path']]}))" >> $O/rect_minb_ab.jsonl
    done
  done
done
unset BITREV_B200_LIB
