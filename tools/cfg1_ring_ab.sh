# cfg1 (2^20 complex128, L2-flushed): register tiles vs TMA tensor ring with all of an SM's tiles in flight
O=gpurun_out
: > $O/cfg1_ring_ab.jsonl
for r in 1 2; do
  for cfg in "def 0 -1" "96 5 2" "96 6 2" "200 5 2" "200 6 2" "200 5 1" "200 4 2"; do
    set -- $cfg
    if [ $1 = def ]; then LIBV=""; else LIBV=variants/lib_ring$1.so; fi
    if [ $1 = 96 ]; then LIBV=""; fi
    env ${LIBV:+BITREV_B200_LIB=$LIBV} python bench.py --workload cfg1 --steps 50 --no-cpu-baseline --no-e2e --tile-bits $2 --tile-path $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'budget': '$1', 'q': $2, 'path': $3, 'value': d['value'], 'median_us': d['step_ms']['median']*1e3, 'l2hot': d['l2_hot']['value'], 'used': [d['config']['tile_bits'], d['config']['tile_path']]}))" >> $O/cfg1_ring_ab.jsonl
  done
done
