timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_hcwb.py -q -x > gpurun_out/s74_pytest.log 2>&1; tail -2 gpurun_out/s74_pytest.log
timeout 300 python bench.py --no-findbest --no-cpu-baseline > gpurun_out/s74_bench.json 2> gpurun_out/s74_bench.err
timeout 300 python bench.py --no-findbest --no-cpu-baseline >> gpurun_out/s74_bench.json 2>> gpurun_out/s74_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s74_launches.csv python bench.py --steps 3 --warmup 3 --no-findbest --no-cpu-baseline > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/s74_launches.csv > gpurun_out/s74_launch_summary.txt 2>&1
