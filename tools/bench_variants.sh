# bench lines of the variants (ACWB, Bernoulli, R2, R2 unbinned, R3, R3 unbinned) -> gpurun_out/m1_bench.log
python __graft_entry__.py build > gpurun_out/m1_build.log 2>&1
for a in "--config R1" "--config R1 --algo acwb" "--config R1 --algo bernoulli" "--config R2" "--config R2 --unbinned" "--config R3 --steps 3" "--config R3 --steps 3 --unbinned"; do
  echo "== $a" >> gpurun_out/m1_bench.log
  timeout 600 python bench.py $a --warmup 3 --no-cpu-baseline >> gpurun_out/m1_bench.log 2>&1
done
