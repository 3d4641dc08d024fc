# round 2, call ar: ncu of k_accum_large at C5
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k "regex:k_accum_large" -c 1 -o gpurun_out/r2ar_accum python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --no-sort --reps 1 --iters 1 > gpurun_out/r2ar_ncu.log 2>&1
