#!/bin/bash
# Full GPU evidence pass (run under gpurun): smoke, GPU tests, bench on every
# workload, reference arm, ncu launch list + full captures of the dominant
# kernels.  Outputs land in gpurun_out/.
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
: > $O/bench_all.jsonl
for w in cfg1 cfg3-4 cfg3-8 cfg3-16 cfg4 cfg4-fft7; do
  python bench.py --workload $w --steps 20 >> $O/bench_all.jsonl 2>> $O/bench_all.err
done
python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_ref.json 2>&1
# ncu: launch list of the default bench, then one full capture per dominant kernel
P="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-soak"
python bench.py $P > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
      --log-file $O/launches_cfg2.csv python bench.py $P > $O/ncu_launch.log 2>&1
for spec in "cfg2:bitrev_" "cfg3-16:bitrev_" "cfg3-4:bitrev_" "cfg3-8:bitrev_" "cfg4:bitrev_" "cfg4-fft7:bitrev_" "cfg1:bitrev_"; do
  w=${spec%%:*}; k=${spec#*:}
  python bench.py --workload $w $P > $O/plain_$w.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
        -o $O/prof_$w python bench.py --workload $w $P > $O/ncu_$w.log 2>&1
  # gpurun copies back <= 64 MiB: keep the raw page of every capture, and the
  # full report of the headline kernel only
  ncu -i $O/prof_$w.ncu-rep --page raw --csv > $O/prof_${w}_raw.csv 2>/dev/null
  [ "$w" = cfg2 ] || rm -f $O/prof_$w.ncu-rep
done
echo gpu_round done
