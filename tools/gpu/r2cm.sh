# round 2, call cm: heavy tiles -- a one-point slot written by its lane (no butterfly)
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or C5 or large_k or k_sweep or dominant or deterministic or configs" > gpurun_out/r2cm_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2cm_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or C5 or large_k" > gpurun_out/r2cm_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2cm_checked.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_hsg0.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_hsg0.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_hsg0.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2cm_sweep.txt 2>&1
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_assign_heavy' -c 20 --csv --log-file gpurun_out/r2cm_launches.csv python bench.py --workload C5 --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2cm_ncu.log 2>&1
KMEANS_LIB_OVERRIDE=paper_2405_12052_b200/libkmeans.so timeout -s KILL 300 python tools/ab_bitwise.py dump gpurun_out/r2cm_ab_new.npz > gpurun_out/r2cm_ab.txt 2>&1
KMEANS_LIB_OVERRIDE=tune/libkmeans_htold.so timeout -s KILL 300 python tools/ab_bitwise.py dump gpurun_out/r2cm_ab_old.npz >> gpurun_out/r2cm_ab.txt 2>&1
python tools/ab_bitwise.py compare gpurun_out/r2cm_ab_new.npz gpurun_out/r2cm_ab_old.npz >> gpurun_out/r2cm_ab.txt 2>&1
KMEANS_LIB_OVERRIDE=tune/libkmeans_hprof.so timeout -s KILL 300 python tools/sweep.py tune/libkmeans_hprof.so --workload C5 --reps 1 > gpurun_out/r2cm_prof.txt 2>&1
