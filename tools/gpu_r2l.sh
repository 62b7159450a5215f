# Round-2 batch: host-buffer paths (pipeline, numpy, concurrency) parity and e2e lines.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_capi_ctypes.py tests/test_gpu_concurrency.py tests/test_gpu_golden.py tests/test_gpu_parity.py -m gpu -q -x -k "host or pipeline or numpy or concurren or ctypes" > $O/pytest_host.log 2>&1; echo pytest=$?; tail -2 $O/pytest_host.log
python bench.py --no-cpu-baseline --no-sweep > $O/bench_e2e.json 2>&1; echo bench=$?
python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_e2e_cfg2.json 2>&1; echo bench2=$?
