timeout 600 python -m pytest tests/test_gpu_degree.py tests/test_gpu_parity.py -q -x -k "limit or pool or bin" > gpurun_out/s78_pytest.log 2>&1; tail -3 gpurun_out/s78_pytest.log
