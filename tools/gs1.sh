timeout 900 python -m pytest tests/test_gpu_acwb.py tests/test_gpu_hcwb.py -x -q > gpurun_out/s53_pytest.log 2>&1; tail -3 gpurun_out/s53_pytest.log
for a in acwb hcwb; do
  timeout 300 python bench.py --algo $a --steps 10 --warmup 3 > gpurun_out/s53_bench_$a.json 2> gpurun_out/s53_bench_$a.err
done
CWB_ACC_T=256 timeout 120 python tools/phase_timing.py R1 256 acwb > gpurun_out/s53_phase.log 2>&1
timeout 120 python tools/phase_timing.py R1 256 acwb >> gpurun_out/s53_phase.log 2>&1
timeout 120 python tools/phase_timing.py R1 256 hcwb >> gpurun_out/s53_phase.log 2>&1
