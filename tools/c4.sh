timeout 600 python tools/gram_timing.py R1 R2 R3 R4 > gpurun_out/c4_gram_timing.log 2>&1
BENCH_ALLOW_SHORT=1 timeout 300 python tools/prof_iter.py R3 1 > gpurun_out/c4_plain.log 2>&1 && timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_h1 -s 1 -c 1 -o gpurun_out/c4_h1_R3 python tools/prof_iter.py R3 1 > gpurun_out/c4_ncu.log 2>&1
