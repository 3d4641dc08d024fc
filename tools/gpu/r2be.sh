# round 2, call be: 3-4 candidate chunks with register sums (large K)
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or ragged or dominant or deterministic or full_size or persist" > gpurun_out/r2be_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2be_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_fewc0.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_fewc0.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2be_sweep.txt 2>&1
done
