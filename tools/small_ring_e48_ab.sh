#!/bin/bash
# float64 / float32 arrays at the <= 32 MiB tiers: register tiles (the tier
# default) against TMA tensor rings with 256-byte rows (E=8 Q5, E=4 Q6) and
# the tier's own width, L2-flushed and L2-resident.
O=gpurun_out
: > $O/small_ring_e48_ab.jsonl
for r in 1 2; do
  python tools/small_ring_probe.py --tag 96 --E 8 --bits 20 21 22 --cands 4:0 4:2 5:2 >> $O/small_ring_e48_ab.jsonl
  python tools/small_ring_probe.py --tag 96 --E 4 --bits 21 22 23 --cands 5:0 5:2 6:2 >> $O/small_ring_e48_ab.jsonl
done
