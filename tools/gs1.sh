timeout 600 python -m pytest tests/test_gpu_bernoulli.py tests/test_gpu_folds.py -x -q > gpurun_out/s51_pytest.log 2>&1; tail -3 gpurun_out/s51_pytest.log
timeout 120 python tools/phase_timing.py R1 256 bernoulli > gpurun_out/s51_phase.log 2>&1
timeout 300 python bench.py --algo bernoulli --steps 10 --warmup 3 > gpurun_out/s51_bench_bern.json 2> gpurun_out/s51_bench_bern.err
