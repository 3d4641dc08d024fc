# round 2, call ab: 512-point chunks (sct4) at C5 and the shards
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_sct4.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2ab_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2ab_sweep.txt 2>&1
done
