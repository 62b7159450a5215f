#!/bin/bash
# Small arrays: register tiles vs the TMA tensor ring at 96 KB and 200 KB
# ring budgets (tools/small_ring_probe.py), two interleaved rounds.
O=gpurun_out
: > $O/small_ring_ab.jsonl
for r in 1 2; do
  python tools/small_ring_probe.py --tag 96 >> $O/small_ring_ab.jsonl
  BITREV_B200_LIB=variants/lib_ring200.so python tools/small_ring_probe.py --tag 200 >> $O/small_ring_ab.jsonl
done
