set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1_smi.txt 2>&1
timeout 600 python tools/peaks.py gpurun_out/peaks_fp64.json > gpurun_out/c1_peaks.log 2>&1
timeout 900 python bench.py --config R3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c1_bench_R3.json 2> gpurun_out/c1_bench_R3.err
timeout 900 python bench.py --config R4 --steps 3 --warmup 3 --no-cpu-baseline --no-findbest > gpurun_out/c1_bench_R4.json 2> gpurun_out/c1_bench_R4.err
