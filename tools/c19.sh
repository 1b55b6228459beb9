timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_jitter.py tests/test_gpu_errors.py -q -x > gpurun_out/c19_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c19_pytest.log
for CFG in R2 R3 R4; do python tools/findbest_timing.py $CFG 1 20 0 1 >> gpurun_out/c19_fb.log 2>&1; done
for CFG in R3 R4; do CWB_STREAM_NOFIT=1 python tools/findbest_timing.py $CFG 1 20 0 1 | sed 's/^/NOFIT /' >> gpurun_out/c19_fb.log 2>&1; done
