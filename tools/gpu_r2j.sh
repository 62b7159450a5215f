# Round-2 batch: auxiliary kernels (transpose, even-odd) parity and GB/s.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_aux_kernels.py tests/test_gpu_golden.py tests/test_gpu_capi_ctypes.py tests/test_gpu_concurrency.py -m gpu -q -x -k "aux or transpose or even_odd or pipeline or concurren or ctypes or every_width or strided" > $O/pytest_aux.log 2>&1; echo pytest=$?; tail -2 $O/pytest_aux.log
timeout 300 python tools/aux_kernels_gbs.py > $O/aux_gbs.json 2>&1; cat $O/aux_gbs.json
