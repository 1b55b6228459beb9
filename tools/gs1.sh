timeout 400 python bench.py > gpurun_out/s69_bench.json 2> gpurun_out/s69_bench.err; tail -3 gpurun_out/s69_bench.err
