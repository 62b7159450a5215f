#!/bin/bash
# complex128 arrays of 2^17..2^21 (the <= 32 MiB tier): register Q5 (default)
# against TMA tensor rings at Q4 / Q5 with 96 KB (default build) and 200 KB
# (variants/lib_ring200.so) budgets, L2-flushed and L2-resident.
O=gpurun_out
: > $O/small_ring_e16_ab.jsonl
for r in 1 2; do
  python tools/small_ring_probe.py --tag 96 --E 16 --bits 17 18 19 20 21 --cands 5:0 4:2 5:2 >> $O/small_ring_e16_ab.jsonl
  BITREV_B200_LIB=variants/lib_ring200.so python tools/small_ring_probe.py --tag 200 --E 16 --bits 17 18 19 20 21 --cands 4:2 5:2 >> $O/small_ring_e16_ab.jsonl
done
