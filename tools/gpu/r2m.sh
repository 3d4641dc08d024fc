# round 2, call m: heavy kernel v2 (warp per sub-tile, no block barriers until the row) + large-K pruned v2
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2m_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2m_gputest.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or large_k or k_sweep or C5" > gpurun_out/r2m_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2m_checked.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_lmb16.so tune/libkmeans_lmb24.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2m_sweep.txt 2>&1
done
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "full_size_c5" > gpurun_out/r2m_c5full.txt 2>&1; echo "rc=$?" >> gpurun_out/r2m_c5full.txt
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_c5_launches.csv python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --reps 5 --iters 3 > gpurun_out/r2m_launch.log 2>&1
