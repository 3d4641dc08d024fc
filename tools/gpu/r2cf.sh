# round 2, call cf: create-time kernels templated on d (no stack arrays); Morton bits A/B
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "configs or sort or ragged or C5 or full_run or deterministic" > gpurun_out/r2cf_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2cf_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_base.so tune/libkmeans_mx4.so; do
  for w in NS C5; do
    echo "== $lib $w" >> gpurun_out/r2cf_e2e.txt
    KMEANS_LIB_OVERRIDE=$lib KMEANS_TRACE=1 timeout -s KILL 600 python tools/e2e_profile.py --workload $w --reps 2 >> gpurun_out/r2cf_e2e.txt 2>&1
  done
done
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_mx4.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2cf_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib >> gpurun_out/r2cf_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2cf_sweep.txt 2>&1
done
