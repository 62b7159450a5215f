#!/bin/bash
# ring-depth A/B across build variants (under gpurun)
out=${1:-gpurun_out/ring_variants.jsonl}
: > $out
for lib in paper_1708_01873_b200/libbitrev_sm100a.so variants/lib_ring*.so; do
  for cfg in "inplace 26 8 5 2" "inplace 26 8 6 2" "inplace 26 16 5 2" "inplace 26 16 4 2" "inplace 26 4 6 2" "oop 26 8 5 2" "oop 26 8 6 1" "oop 26 16 5 1" "oop 26 16 4 1"; do
    echo "{\"lib\": \"$lib\"}" >> $out
    BITREV_B200_LIB=$lib python tools/order_sweep.py $cfg 0 >> $out 2>&1
  done
done
