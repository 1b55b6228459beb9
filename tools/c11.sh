timeout 1200 python -m pytest tests/test_gpu_gram.py -q -rs -s > gpurun_out/c11_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c11_pytest.log
timeout 600 python tools/gram_timing.py R1 R2 R3 R4 > gpurun_out/c11_gram_timing.log 2>&1
CWB_GRAM_DENSE=1 timeout 600 python tools/gram_timing.py R3 R4 > gpurun_out/c11_gram_timing_dense.log 2>&1
