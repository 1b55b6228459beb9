timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "paths_agree or batch_hint or r2_full or tie_following or r3_full" -s > gpurun_out/c6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c6_pytest.log
CWB_H1_WIDE=0 timeout 300 python tools/gram_timing.py R3 > gpurun_out/c6_gram_narrowh1.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/c6_bench_R3.json 2> gpurun_out/c6_bench_R3.err
CWB_H1_WIDE=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-findbest --no-cpu-baseline --no-gram > gpurun_out/c6_bench_R3_narrow.json 2> gpurun_out/c6_bench_R3_narrow.err
timeout 900 python bench.py --config R4 --steps 3 --warmup 3 --no-findbest --no-cpu-baseline > gpurun_out/c6_bench_R4.json 2> gpurun_out/c6_bench_R4.err
