# round 2, call n: heavy kernel v3 (super list staged in shared memory)
set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or large_k or k_sweep or C5 or 257" > gpurun_out/r2n_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2n_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or large_k" > gpurun_out/r2n_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2n_checked.txt
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 >> gpurun_out/r2n_sweep.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n_c5_launches.csv python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --reps 5 --iters 3 > gpurun_out/r2n_launch.log 2>&1
