# round 2, call cl: large-K pruned prologue keeps the first super-list entry per lane between passes
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or C5 or large_k or k_sweep or dominant or deterministic or configs" > gpurun_out/r2cl_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2cl_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or C5 or large_k" > gpurun_out/r2cl_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2cl_checked.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_pcc0.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_pcc0.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_pcc0.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2cl_sweep.txt 2>&1
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_assign_pruned' -c 20 --csv --log-file gpurun_out/r2cl_launches.csv python bench.py --workload C5 --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2cl_ncu.log 2>&1
