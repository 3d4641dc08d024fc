# round 2, call ci: heavy tiles gathered walk vs not (A/B repeat)
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_hnog.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_hnog.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_hnog.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2ci_sweep.txt 2>&1
done
