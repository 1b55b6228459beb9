timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_bernoulli.py -q -x > gpurun_out/s75_pytest.log 2>&1; tail -2 gpurun_out/s75_pytest.log
timeout 120 python tools/phase_timing.py R1 256 cwb > gpurun_out/s75_phase.log 2>&1
CWB_ZALL=0 timeout 120 python tools/phase_timing.py R1 256 cwb >> gpurun_out/s75_phase.log 2>&1
timeout 120 python tools/phase_timing.py R1 256 bernoulli >> gpurun_out/s75_phase.log 2>&1
timeout 120 python tools/phase_timing.py R2 1024 cwb >> gpurun_out/s75_phase.log 2>&1
CWB_ZALL=0 timeout 120 python tools/phase_timing.py R2 1024 cwb >> gpurun_out/s75_phase.log 2>&1
cat gpurun_out/s75_phase.log
timeout 300 python bench.py --no-findbest --no-cpu-baseline > gpurun_out/s75_bench.json 2> gpurun_out/s75_bench.err
