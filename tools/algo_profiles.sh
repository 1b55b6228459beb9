# bench + ncu brief of the fused kernel in ACWB / HCWB / Bernoulli modes -> gpurun_out/r1g_*
TAG=r1g
mkdir -p gpurun_out
python __graft_entry__.py build > gpurun_out/${TAG}_build.log 2>&1
for a in acwb hcwb bernoulli; do
  timeout 300 python bench.py --algo $a --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_$a.json 2>&1
  BENCH_ALLOW_SHORT=1 timeout 600 ncu --set full --clock-control none -k regex:k_train_fused -s 1 -c 1 -o /tmp/${TAG}_fused_$a python bench.py --algo $a --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_$a.log 2>&1
  python tools/ncu_brief.py /tmp/${TAG}_fused_$a.ncu-rep > gpurun_out/${TAG}_ncu_$a.txt 2>&1
done
