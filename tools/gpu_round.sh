#!/bin/bash
# One GPU session: tests, bench, ncu launch list, full capture of the top kernel.
# usage (from repo root, under gpurun): bash tools/gpu_round.sh TAG [CONFIG]
TAG=${1:-r1}; CFG=${2:-R1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python __graft_entry__.py build > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_${CFG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench_${CFG}.log
