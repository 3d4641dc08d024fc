# round 2, call bt: per-chunk phase times of the heavy kernel at C5
timeout -s KILL 300 python tools/sweep.py tune/libkmeans_hprof.so --workload C5 --reps 1 --iters 1 > gpurun_out/r2bt_hprof.txt 2>&1
