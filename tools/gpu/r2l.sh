# round 2, call l: C5 kernels under ncu (launch list + full capture of the assign kernels)
set -x
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_c5_launches.csv python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --reps 5 --iters 3 > gpurun_out/r2l_launch.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:'k_assign_pruned|k_assign_heavy|k_prune' -s 12 -c 3 -o gpurun_out/r2l_c5 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --reps 2 --iters 3 > gpurun_out/r2l_ncu.log 2>&1
