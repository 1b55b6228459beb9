timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s83_pytest.log 2>&1; tail -3 gpurun_out/s83_pytest.log
