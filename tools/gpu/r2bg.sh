# round 2, call bg: slot sums per TMA unit (8 points per lane) with the transposing butterfly
set -x
KMEANS_LIB_OVERRIDE=tune/libkmeans_aggunit.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or dominant" > gpurun_out/r2bg_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bg_tests.txt
for lib in tune/libkmeans_aggunit.so tune/libkmeans_base.so tune/libkmeans_aggunit.so tune/libkmeans_base.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2bg_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2bg_sweep.txt 2>&1
done
