# Round-2 evidence batch: smoke, baseline-size parity tests, default bench, reference arm, cfg2 line.
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_golden.py -m gpu -q -x > $O/pytest_new.log 2>&1; echo pytest=$?; tail -3 $O/pytest_new.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench=$?
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2>&1; echo cfg2=$?
