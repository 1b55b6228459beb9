timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s71_pytest.log 2>&1; tail -3 gpurun_out/s71_pytest.log
