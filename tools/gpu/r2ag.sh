# round 2, call ag: column-path threshold sweep (C5)
set -x
for rep in 1 2; do
for lib in tune/libkmeans_lcol0.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_lcol5.so tune/libkmeans_lcol6.so tune/libkmeans_lcol8.so tune/libkmeans_lcol12.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2ag_sweep.txt 2>&1
done
done
