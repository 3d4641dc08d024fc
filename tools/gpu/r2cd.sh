# round 2, call cd: per-tile phase times of k_assign_heavy_tiles at C5 (KM_HEAVY_PROF)
set -x
KMEANS_LIB_OVERRIDE=tune/libkmeans_hprof.so timeout -s KILL 300 python tools/sweep.py tune/libkmeans_hprof.so --workload C5 --reps 1 > gpurun_out/r2cd_prof.txt 2>&1
