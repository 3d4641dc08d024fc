# round 2, call t: branch-free Hilbert keys; 2D A/B repeated; create time
set -x
for rep in 1 2; do
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_zcurve.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 >> gpurun_out/r2t_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 --N 12500000 >> gpurun_out/r2t_sweep.txt 2>&1
done
done
timeout -s KILL 300 python tools/e2e_profile.py > gpurun_out/r2t_e2e.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_ns_launches.csv python tools/sweep.py paper_2405_12052_b200/libkmeans.so --reps 5 --iters 3 > gpurun_out/r2t_launch.log 2>&1
