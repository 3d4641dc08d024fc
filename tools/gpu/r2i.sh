# round 2, call i: k_persist_iterate v6 (contiguous unit ranges, no predicates) + the no-wait timing experiment
set -x
timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent" > gpurun_out/r2i_persist_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2i_persist_tests.txt
for N in 12500000 100000000; do
  for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_pw20.so tune/libkmeans_pnw.so tune/libkmeans_pnw20.so; do
    timeout -s KILL 300 python tools/sweep.py $lib --N $N >> gpurun_out/r2i_sweep.txt 2>&1
  done
done
