timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/c8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c8_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c8_bench_R3.json 2> gpurun_out/c8_bench_R3.err
timeout 900 python bench.py --config R4 --steps 3 --warmup 3 --no-findbest --no-cpu-baseline --no-gram > gpurun_out/c8_bench_R4.json 2> gpurun_out/c8_bench_R4.err
