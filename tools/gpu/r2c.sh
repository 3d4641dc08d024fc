# round 2, call c: the persistent sorted iteration (k_persist_iterate): parity first, then timing
set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent" > gpurun_out/r2c_persist_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_persist_tests.txt
grep -q "rc=0" gpurun_out/r2c_persist_tests.txt || exit 0
for N in 12500000 25000000 50000000 100000000; do
  timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N $N >> gpurun_out/r2c_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N $N --no-persist >> gpurun_out/r2c_sweep.txt 2>&1
done
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C3 >> gpurun_out/r2c_sweep.txt 2>&1
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C3 --N 12500000 >> gpurun_out/r2c_sweep.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_gputest.txt
