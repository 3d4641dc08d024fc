# round 2, call al: k_assign_large variants (12 points per lane, unroll 2, 4 points per lane)
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_lnpl3.so tune/libkmeans_lu2.so tune/libkmeans_lnpl1.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --reps 5 --iters 2 >> gpurun_out/r2al_sweep.txt 2>&1
  for K in 64 128 400; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --K $K --N 20000000 --reps 10 --iters 2 >> gpurun_out/r2al_sweep.txt 2>&1
  done
done
KMEANS_LIB_OVERRIDE=tune/libkmeans_lnpl3.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or dominant or configs" > gpurun_out/r2al_tests_lnpl3.txt 2>&1; echo "rc=$?" >> gpurun_out/r2al_tests_lnpl3.txt
