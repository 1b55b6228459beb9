timeout 240 python -m pytest tests/test_gpu_clamp.py -q -x > gpurun_out/s58_pytest.log 2>&1 || { echo "clamp rc=$?"; tail -30 gpurun_out/s58_pytest.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_degree.py -q -x >> gpurun_out/s58_pytest.log 2>&1; tail -3 gpurun_out/s58_pytest.log
