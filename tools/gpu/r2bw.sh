# round 2, call bw: heavy refinement unroll x4 vs the committed tree, same box
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_base.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_base.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_base.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2bw_sweep.txt 2>&1
done
