for t in 1024 512 256; do for c in R3 R4; do CWB_FIT_T=$t timeout 180 python tools/findbest_timing.py $c 1 20 0 1 | sed "s/^/T=$t /" >> gpurun_out/s76_fb.log 2>&1; done; done
CWB_FIT_T=256 timeout 300 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/s76_pytest.log 2>&1; tail -1 gpurun_out/s76_pytest.log
cat gpurun_out/s76_fb.log
