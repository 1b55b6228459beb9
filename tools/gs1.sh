timeout 600 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/s67_pytest.log 2>&1; tail -2 gpurun_out/s67_pytest.log
for c in R3 R4 R3 R4; do timeout 120 python tools/findbest_timing.py $c 1 3 0 >> gpurun_out/s67_fb.log 2>&1; done; cat gpurun_out/s67_fb.log
