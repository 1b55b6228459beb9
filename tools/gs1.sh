timeout 600 python -m pytest tests/test_gpu_edges.py -q > gpurun_out/s80_pytest.log 2>&1; tail -30 gpurun_out/s80_pytest.log
