# Round-2 batch: pack/unpack parity, cfg5 phases, cfg2 lines around the tile-swap and run-length probes.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -m gpu -q -x -k "unpack or pack or cfg5" > $O/pytest_pack.log 2>&1; echo pytest=$?; tail -2 $O/pytest_pack.log
timeout 600 python tools/cfg5_phases.py > $O/cfg5_phases2.jsonl 2>&1; echo phases=$?
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2_c.json 2>&1; echo cfg2=$?
timeout 300 ./tools/probe/tileswap > $O/tileswap.jsonl 2>&1; echo tileswap=$?
timeout 300 ./tools/probe/runs > $O/runs_probe2.jsonl 2>&1; echo runs=$?
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2_d.json 2>&1; echo cfg2=$?
