# round 2, call af: large K per-lane columns for <= 4-candidate chunks
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or ragged or scales or bisector" > gpurun_out/r2af_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2af_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or heavy or large_k or C5" > gpurun_out/r2af_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2af_checked.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_lcol0.so tune/libkmeans_lcol6.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2af_sweep.txt 2>&1
done
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "full_size_c5" > gpurun_out/r2af_c5full.txt 2>&1; echo "rc=$?" >> gpurun_out/r2af_c5full.txt
