# round 2, call am: split large-K full scan (labels pass + k_accum_large) vs fused
set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or extreme or configs or deterministic or dominant or full_run or fake_sharding or profile_stages" > gpurun_out/r2am_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2am_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_lsplit64.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or dominant or configs" > gpurun_out/r2am_tests_split64.txt 2>&1; echo "rc=$?" >> gpurun_out/r2am_tests_split64.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_lnosplit.so tune/libkmeans_lsnpl1.so tune/libkmeans_lsnpl3.so tune/libkmeans_lsplit64.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --reps 5 --iters 2 >> gpurun_out/r2am_sweep.txt 2>&1
  for K in 64 200 400 600; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --K $K --N 20000000 --reps 10 --iters 2 >> gpurun_out/r2am_sweep.txt 2>&1
  done
done
