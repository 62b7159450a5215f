# Round-2 batch: benchmark-API tests, DRAM run-length probe, cfg5 local phases, cfg5 on one GPU.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_api.py -m gpu -q -x > $O/pytest_api.log 2>&1; echo pytest=$?; tail -3 $O/pytest_api.log
timeout 300 ./tools/probe/runs > $O/runs_probe.jsonl 2>&1; echo runs=$?
timeout 600 python tools/cfg5_phases.py > $O/cfg5_phases.jsonl 2>&1; echo phases=$?
timeout 300 python bench.py --workload cfg5 --steps 5 --no-cpu-baseline > $O/bench_cfg5_n1.json 2>&1; echo cfg5n1=$?
