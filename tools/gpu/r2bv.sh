# round 2, call bv: heavy-kernel refinement loops unrolled x4 only
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or dominant or full_size or deterministic or ragged" > gpurun_out/r2bv_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bv_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_ru1.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_ru1.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2bv_sweep.txt 2>&1
done
