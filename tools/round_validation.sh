# round-end validation on one B200 (run under gpurun from the repo root): tests, smoke, bench (plain and
# torchrun N=1), reference arm, launch list and an ncu capture of the top kernel -> gpurun_out/${TAG}_*
# usage: /usr/local/graft/bin/gpurun --timeout 3000 -- 'TAG=r1z bash tools/round_validation.sh'
TAG=${TAG:-r1z}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gpu_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 400 python bench.py > gpurun_out/${TAG}_bench_R1.json 2> gpurun_out/${TAG}_bench_R1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_torchrun.json 2> gpurun_out/${TAG}_bench_torchrun.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref_R1.json 2> gpurun_out/${TAG}_ref_R1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_R1.csv python bench.py --steps 3 --warmup 3 --no-findbest --no-cpu-baseline > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/${TAG}_launches_R1.csv > gpurun_out/${TAG}_launches_R1_summary.txt 2>&1
BENCH_ALLOW_SHORT=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_train_fused -s 1 -c 1 -o /tmp/${TAG}_fused python bench.py --steps 1 --warmup 1 --no-findbest --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_brief.py /tmp/${TAG}_fused.ncu-rep > gpurun_out/${TAG}_ncu_fused_R1.txt 2>&1
