python __graft_entry__.py build > gpurun_out/s11_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hcwb.py tests/test_gpu_acwb.py -x -q > gpurun_out/s11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s11_pytest.log
timeout 300 python bench.py --algo hcwb --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s11_bench_hcwb.log 2>&1
