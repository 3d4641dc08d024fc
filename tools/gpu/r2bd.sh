# round 2, call bd: candidate-count histogram at C5 and NS shards
KMEANS_TRACE=1 timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --reps 5 > gpurun_out/r2bd_hist.txt 2>&1
KMEANS_TRACE=1 timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N 12500000 --reps 5 >> gpurun_out/r2bd_hist.txt 2>&1
