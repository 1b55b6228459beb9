timeout 1500 python -m pytest tests/test_gpu_gram.py tests/test_gpu_jitter.py tests/test_gpu_errors.py tests/test_gpu_hcwb.py -q -rs -s > gpurun_out/c5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c5_pytest.log
timeout 600 python tools/gram_timing.py R1 R2 R3 R4 > gpurun_out/c5_gram_timing.log 2>&1
