# complex128 Q5 tier at 1 vs 4 CTAs/SM over b = 17..21 (size curve), then the pack shared-memory A/B.
O=gpurun_out
: > $O/minb_sizes_ab.jsonl
for r in 1 2; do
  for m in 1 4; do
    BITREV_B200_SMALL_MINB=$m python tools/size_curve.py --bits 17 18 19 20 21 --widths 16 --reps 40 2>/dev/null | sed "s/^{/{\"minb\": $m, /" >> $O/minb_sizes_ab.jsonl
  done
done
bash tools/pack_smem_ab.sh
