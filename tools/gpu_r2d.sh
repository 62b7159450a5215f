# Round-2 batch: sharded parity, cfg5 phases, run-length probe, cfg2 line.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_golden.py -m gpu -q -x -k "unpack or pack or cfg5 or sharded" > $O/pytest_pack2.log 2>&1; echo pytest=$?; tail -2 $O/pytest_pack2.log
timeout 600 python tools/cfg5_phases.py > $O/cfg5_phases3.jsonl 2>&1; echo phases=$?
timeout 300 ./tools/probe/runs > $O/runs_probe3.jsonl 2>&1; echo runs=$?
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2_e.json 2>&1; echo cfg2=$?
