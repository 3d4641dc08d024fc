# round 2, call e: k_persist_iterate v3 (per-warp tables, block + grid last-arriver merge)
set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent" > gpurun_out/r2e_persist_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2e_persist_tests.txt
grep -q "rc=0" gpurun_out/r2e_persist_tests.txt || exit 0
for N in 12500000 25000000 100000000; do
  for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_pw24.so tune/libkmeans_pw20.so; do
    timeout -s KILL 300 python tools/sweep.py $lib --N $N >> gpurun_out/r2e_sweep.txt 2>&1
  done
  timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N $N --no-persist >> gpurun_out/r2e_sweep.txt 2>&1
done
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C3 --N 12500000 >> gpurun_out/r2e_sweep.txt 2>&1
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C3 >> gpurun_out/r2e_sweep.txt 2>&1
