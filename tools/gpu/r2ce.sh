# round 2, call ce: k_assign_heavy_tiles with slot sums spread over the warps and split walks from 8 entries
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or dominant or deterministic or ragged" > gpurun_out/r2ce_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ce_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_htold.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_htold.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2ce_sweep.txt 2>&1
done
KMEANS_LIB_OVERRIDE=tune/libkmeans_hprof.so timeout -s KILL 300 python tools/sweep.py tune/libkmeans_hprof.so --workload C5 --reps 1 > gpurun_out/r2ce_prof.txt 2>&1
