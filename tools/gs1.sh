timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fit_host" > gpurun_out/s84_pytest.log 2>&1; tail -1 gpurun_out/s84_pytest.log
for i in 1 2; do timeout 300 python bench.py --no-findbest --no-cpu-baseline >> gpurun_out/s84_bench.json 2>> gpurun_out/s84_bench.err; done
