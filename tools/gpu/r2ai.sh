# round 2, call ai: k_assign_large step shapes (points per lane x centroids per step)
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_l4k8.so tune/libkmeans_l4k16.so tune/libkmeans_l8k16.so; do
  KMEANS_LIB_OVERRIDE=$lib timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or extreme" > gpurun_out/r2ai_tests_$(basename $lib .so).txt 2>&1; echo "rc=$?" >> gpurun_out/r2ai_tests_$(basename $lib .so).txt
done
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_l4k8.so tune/libkmeans_l4k16.so tune/libkmeans_l8k16.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --reps 5 --iters 2 >> gpurun_out/r2ai_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --K 64 --N 20000000 --reps 10 --iters 2 >> gpurun_out/r2ai_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --K 200 --N 20000000 --reps 10 --iters 2 >> gpurun_out/r2ai_sweep.txt 2>&1
done
