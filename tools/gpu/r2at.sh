# round 2, call at: full-scan K<=16 three-stage tile pipeline (cpipe) A/B
set -x
for lib in tune/libkmeans_cpipe.so tune/libkmeans_cpipe8.so; do
KMEANS_LIB_OVERRIDE=$lib timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or configs" > gpurun_out/r2at_tests_$(basename $lib .so).txt 2>&1; echo "rc=$?" >> gpurun_out/r2at_tests_$(basename $lib .so).txt
done
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_cpipe.so tune/libkmeans_cpipe9.so tune/libkmeans_cpipe8.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --no-sort --reps 20 --iters 2 >> gpurun_out/r2at_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 --no-sort --reps 20 --iters 2 >> gpurun_out/r2at_sweep.txt 2>&1
done
