nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c2_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/c2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/c2_bench_R3.json 2> gpurun_out/c2_bench_R3.err
timeout 300 python tools/prof_iter.py R3 3 > gpurun_out/c2_prof.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches_R3.csv python tools/prof_iter.py R3 3 > /dev/null 2>&1
