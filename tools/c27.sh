CWB_H1_X4=1 CWB_H1_CHUNK_MB=20 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c27_R3_x4_20.json 2> gpurun_out/c27.err
CWB_H1_X4=1 CWB_H1_CHUNK_MB=12 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c27_R3_x4_12.json 2>> gpurun_out/c27.err
