# round 2, call an: large-K defaults (split below 8 fused warps, 12 points per lane) across K
set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or dominant or configs or deterministic" > gpurun_out/r2an_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2an_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_lnosplit.so tune/libkmeans_lnb2.so tune/libkmeans_lsplit12.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --reps 5 --iters 2 >> gpurun_out/r2an_sweep.txt 2>&1
  for K in 500 600 800; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 --no-sort --K $K --N 20000000 --reps 10 --iters 2 >> gpurun_out/r2an_sweep.txt 2>&1
  done
done
