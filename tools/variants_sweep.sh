#!/bin/bash
# A/B the build variants in variants/ on the GPU (called under gpurun).
set -u
out=${1:-gpurun_out/variants.jsonl}
: > $out
for lib in paper_1708_01873_b200/libbitrev_sm100a.so variants/lib_*.so; do
  echo "{\"lib\": \"$lib\"}" >> $out
  BITREV_B200_LIB=$lib python tools/sweep.py --bits 26 30 --widths 8 16 4 --orders 0 --reps 10 >> $out 2>&1
done
