# E=8 in place: register pairs (path 0) vs 2-CTA cluster pairs (path 6) at 256 / 128 threads
# Historical record: the knob this A/B switched was removed from the library after
# the measurement (result under profiles/r02_*); rerunning measures the default twice.
O=gpurun_out
: > $O/ip_cluster_nt_ab.jsonl
for r in 1 2 3; do
  for cfg in "0 256" "6 256" "6 128" "6 129" "6 130"; do
    set -- $cfg
    BITREV_B200_PATH_IP=$1 BITREV_B200_IP_CLUSTER_NT=$2 python bench.py --workload cfg2 --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'path': $1, 'nt': $2, 'value': d['value'], 'tile': [d['config']['tile_bits'], d['config']['tile_path']]}))" >> $O/ip_cluster_nt_ab.jsonl
  done
done
