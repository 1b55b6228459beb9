CWB_H1_CHUNKING=0 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c17_R3_nochunk.json 2>/dev/null
CWB_H1_CHUNK_MB=64 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c17_R3_64.json 2>/dev/null
CWB_H1_CHUNK_MB=24 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c17_R3_24.json 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c17_R3_40.json 2>/dev/null
CWB_H1_CHUNK_MB=64 timeout 900 python bench.py --config R4 --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c17_R4_64.json 2>/dev/null
CWB_H1_CHUNK_MB=24 timeout 900 python bench.py --config R4 --steps 3 --warmup 3 --no-cpu-baseline --no-findbest --no-gram > gpurun_out/c17_R4_24.json 2>/dev/null
