timeout 600 python -m pytest tests/test_gpu_csr.py tests/test_gpu_clamp.py -q -x > gpurun_out/s87_pytest.log 2>&1; tail -2 gpurun_out/s87_pytest.log
timeout 300 python tools/init_timing.py R4 5 > gpurun_out/s87_init.log 2>&1; timeout 300 python tools/init_timing.py R3 5 >> gpurun_out/s87_init.log 2>&1; cat gpurun_out/s87_init.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s87_init_R4.csv python tools/init_timing.py R4 1 > /dev/null 2>&1
