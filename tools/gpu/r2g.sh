# round 2, call g: ncu of k_persist_iterate (pw20 build) at the P=8 NS shard (N = 1.25e7)
set -x
export KMEANS_LIB_OVERRIDE=tune/libkmeans_pw20.so
timeout -s KILL 120 python tools/persist_probe.py --N 12500000 --iters 20 > gpurun_out/r2g_probe.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_persist -c 1 -o gpurun_out/r2g_persist python tools/persist_probe.py --N 12500000 --iters 20 > gpurun_out/r2g_ncu.log 2>&1
unset KMEANS_LIB_OVERRIDE
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_pruned -c 1 -o gpurun_out/r2g_pruned python tools/persist_probe.py --N 12500000 --iters 3 --no-persist > gpurun_out/r2g_ncu2.log 2>&1
