CWB_H1_X4=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c26_R3_x4.json 2> gpurun_out/c26_R3_x4.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c26_R3_x2.json 2> gpurun_out/c26_R3_x2.err
