# round 2, call ad: row-group size (k_merge_sparse16 rows per group) re-check
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_rg512.so tune/libkmeans_rg1024.so; do
  for N in 12500000 25000000 100000000; do
    timeout -s KILL 300 python tools/sweep.py $lib --N $N >> gpurun_out/r2ad_sweep.txt 2>&1
  done
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 >> gpurun_out/r2ad_sweep.txt 2>&1
done
