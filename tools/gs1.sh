python __graft_entry__.py build > gpurun_out/s20_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -x -q -k "stream or find_best" > gpurun_out/s20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s20_pytest.log
for cfg in R2 R3 R4; do timeout 120 python tools/findbest_timing.py $cfg 1 20 0 >> gpurun_out/s20_fb.log 2>&1; done
timeout 120 python tools/findbest_timing.py R4 2 20 0 >> gpurun_out/s20_fb.log 2>&1
timeout 120 python tools/findbest_timing.py R3 4 20 0 >> gpurun_out/s20_fb.log 2>&1
timeout 120 python tools/findbest_timing.py R4 1 3 0 > gpurun_out/s20_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_h1_stream" -s 1 -c 1 -o gpurun_out/s20_stream python tools/findbest_timing.py R4 1 3 0 > gpurun_out/s20_ncu.log 2>&1
