# round 2, call bz: large-K pruned kernel in reverse chunk order
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or dominant or full_size or deterministic or persist or ragged" > gpurun_out/r2bz_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bz_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_lfwd.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_lfwd.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2bz_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2bz_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib >> gpurun_out/r2bz_sweep.txt 2>&1
done
