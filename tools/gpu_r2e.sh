# Round-2 batch: ncu captures of the cfg5 pack/unpack, cfg2 and cfg3-16, and the default launch list.
set -u
O=gpurun_out
python tools/ncu_cfg5.py > $O/ncu_cfg5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pack_rect|sharded_unpack" -s 2 -c 2 -o $O/prof_cfg5 python tools/ncu_cfg5.py > $O/ncu_cfg5.log 2>&1
ncu -i $O/prof_cfg5.ncu-rep --page raw --csv > $O/prof_cfg5_raw.csv 2>/dev/null
rm -f $O/prof_cfg5.ncu-rep
python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-soak > $O/plain_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bitrev_ -s 3 -c 1 -o $O/prof_cfg2 python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-soak > $O/ncu_cfg2.log 2>&1
ncu -i $O/prof_cfg2.ncu-rep --page raw --csv > $O/prof_cfg2_raw.csv 2>/dev/null
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-soak --no-sweep > $O/plain_cfg316.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_cfg316.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-soak --no-sweep > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bitrev_ -s 3 -c 1 -o $O/prof_cfg316 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-soak --no-sweep > $O/ncu_cfg316.log 2>&1
ncu -i $O/prof_cfg316.ncu-rep --page raw --csv > $O/prof_cfg316_raw.csv 2>/dev/null
rm -f $O/prof_cfg316.ncu-rep
echo done
