#!/bin/bash
# Full GPU evidence pass (run under gpurun): smoke, GPU tests, the default
# bench line (cfg3-16 + width sweep), every other workload, the reference arm,
# ncu launch list of the default bench and one full capture per dominant
# kernel.  Outputs land in gpurun_out/.
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err
: > $O/bench_all.jsonl
for w in cfg1 cfg2 cfg4 cfg4-fft7; do
  python bench.py --workload $w --steps 20 >> $O/bench_all.jsonl 2>> $O/bench_all.err
done
python bench.py --workload cfg5 --steps 5 --no-cpu-baseline >> $O/bench_all.jsonl 2>> $O/bench_all.err
python bench.py --impl reference > $O/bench_ref.json 2>&1
python bench.py --impl reference --workload cfg2 >> $O/bench_ref.json 2>&1
# ncu: launch list of the default bench, then one full capture per dominant kernel
P="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-soak --no-sweep"
python bench.py $P > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file $O/launches_default.csv python bench.py $P > $O/ncu_launch.log 2>&1
for w in cfg3-16 cfg3-4 cfg3-8 cfg2 cfg4 cfg4-fft7 cfg1; do
  python bench.py --workload $w $P > $O/plain_$w.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:bitrev_ -s 3 -c 1 \
        -o $O/prof_$w python bench.py --workload $w $P > $O/ncu_$w.log 2>&1
  ncu -i $O/prof_$w.ncu-rep --page raw --csv > $O/prof_${w}_raw.csv 2>/dev/null
  rm -f $O/prof_$w.ncu-rep
done
echo gpu_round done
