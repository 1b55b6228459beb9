# round-end validation on one B200 (run under gpurun from the repo root): tests, smoke, bench (plain and
# torchrun N=1), reference arm, launch list and an ncu capture of the top kernel -> gpurun_out/${TAG}_*
# usage: /usr/local/graft/bin/gpurun --timeout 3600 -- 'TAG=r2z bash tools/round_validation.sh'
TAG=${TAG:-r2z}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/${TAG}_gpu_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gpu_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_R3.json 2> gpurun_out/${TAG}_bench_R3.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_torchrun.json 2> gpurun_out/${TAG}_bench_torchrun.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref_R3.json 2> gpurun_out/${TAG}_ref_R3.err
timeout 600 python bench.py --config R1 --steps 10 --warmup 3 --no-gram > gpurun_out/${TAG}_bench_R1.json 2> gpurun_out/${TAG}_bench_R1.err
timeout 900 python bench.py --config R4 --steps 3 --warmup 3 --no-findbest --no-cpu-baseline > gpurun_out/${TAG}_bench_R4.json 2> gpurun_out/${TAG}_bench_R4.err
BENCH_ALLOW_SHORT=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_R3.csv python bench.py --steps 1 --warmup 1 --no-findbest --no-cpu-baseline --no-gram > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/${TAG}_launches_R3.csv > gpurun_out/${TAG}_launches_R3_summary.txt 2>&1
timeout 300 python tools/prof_iter.py R3 1 > gpurun_out/${TAG}_prof_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_h1w -s 2 -c 1 -o gpurun_out/${TAG}_h1w python tools/prof_iter.py R3 1 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_brief.py gpurun_out/${TAG}_h1w.ncu-rep > gpurun_out/${TAG}_ncu_h1w_R3.txt 2>&1
# DRAM bytes of the H1 phase of one R3 iteration (its row-chunk launches), for roofline.traffic (profiles/traffic.json)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_h1w -c 6 --csv --log-file gpurun_out/${TAG}_h1w_traffic.csv python tools/prof_iter.py R3 1 > /dev/null 2>&1
# R1 variants of the fused kernel (ACWB, HCWB, Bernoulli) and the findBest B = 1 split
for a in acwb hcwb bernoulli; do timeout 600 python bench.py --config R1 --algo $a --steps 10 --warmup 3 --no-gram --no-cpu-baseline --no-findbest > gpurun_out/${TAG}_bench_R1_$a.json 2> gpurun_out/${TAG}_bench_R1_$a.err; done
for cfg in R3 R4; do timeout 300 python tools/findbest_timing.py $cfg 1 20 0 1 >> gpurun_out/${TAG}_findbest.log 2>&1; CWB_STREAM_NOFIT=1 timeout 300 python tools/findbest_timing.py $cfg 1 20 0 1 | sed 's/^/NOFIT /' >> gpurun_out/${TAG}_findbest.log 2>&1; done
