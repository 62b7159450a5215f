# pack kernel occupancy A/B (G = 8 shard): default (3 CTAs/SM) vs 2 CTAs/SM (80 KB smem)
O=gpurun_out
: > $O/pack_smem_ab.jsonl
for r in 1 2 3; do
  for kb in 0 80; do
    BITREV_B200_PACK_SMEM_KB=$kb python tools/cfg5_phases.py 2>/dev/null | grep pack_k4 | sed "s/^{/{\"smem_kb\": $kb, /" >> $O/pack_smem_ab.jsonl
  done
done
