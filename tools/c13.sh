for LD in 0 1 2; do
CWB_H1_LD=$LD timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c13_bench_R3_ld$LD.json 2> gpurun_out/c13_bench_R3_ld$LD.err
done
CWB_H1_LD=1 timeout 900 python bench.py --config R4 --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c13_bench_R4_ld1.json 2> gpurun_out/c13_bench_R4_ld1.err
