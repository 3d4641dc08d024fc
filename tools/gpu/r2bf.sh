# round 2, call bf: row-merge group size at the strong-scaling shard sizes
set -x
for r in 1 2; do
for lib in tune/libkmeans_base.so tune/libkmeans_rg128.so tune/libkmeans_rg64.so; do
  for N in 12500000 25000000; do
    timeout -s KILL 300 python tools/sweep.py $lib --N $N --reps 300 >> gpurun_out/r2bf_sweep.txt 2>&1
  done
done
done
timeout -s KILL 300 python tools/sweep.py tune/libkmeans_base.so >> gpurun_out/r2bf_sweep.txt 2>&1
timeout -s KILL 300 python tools/sweep.py tune/libkmeans_rg128.so >> gpurun_out/r2bf_sweep.txt 2>&1
