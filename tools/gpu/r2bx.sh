# round 2, call bx: chunks per prune super box (16 / 32 / 64 / 128) at C5
set -x
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_sup16.so tune/libkmeans_sup32.so tune/libkmeans_sup128.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_sup16.so tune/libkmeans_sup32.so tune/libkmeans_sup128.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2bx_sweep.txt 2>&1
done
KMEANS_LIB_OVERRIDE=tune/libkmeans_sup32.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "C5 or heavy or large_k or k_sweep" > gpurun_out/r2bx_tests32.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bx_tests32.txt
