# round 2, call k: large-K pruned kernel v2 (single pass, <= 64-slot table, no per-lane columns)
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2k_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2k_gputest.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_lmb16.so tune/libkmeans_lmb24.so tune/libkmeans_lc32.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2k_sweep.txt 2>&1
done
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so >> gpurun_out/r2k_sweep.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "full_size_c5" > gpurun_out/r2k_c5full.txt 2>&1; echo "rc=$?" >> gpurun_out/r2k_c5full.txt
