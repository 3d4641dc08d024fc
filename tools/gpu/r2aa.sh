# round 2, call aa: heavy tiles with long lists walked by all 8 warps
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs" > gpurun_out/r2aa_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2aa_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or large_k" > gpurun_out/r2aa_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2aa_checked.txt
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 >> gpurun_out/r2aa_sweep.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2aa_c5_launches.csv python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --reps 5 --iters 3 > gpurun_out/r2aa_launch.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "full_size_c5" > gpurun_out/r2aa_c5full.txt 2>&1; echo "rc=$?" >> gpurun_out/r2aa_c5full.txt
