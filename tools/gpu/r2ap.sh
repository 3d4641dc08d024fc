# round 2, call ap: k_accum_large with 4 sub-tiles per warp step
set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or dominant or configs or full_size_c5" > gpurun_out/r2ap_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ap_tests.txt
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --no-sort --reps 5 --iters 2 >> gpurun_out/r2ap_sweep.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k "regex:k_accum_large" -c 2 --csv --log-file gpurun_out/r2ap_accum.csv python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --no-sort --reps 1 --iters 1 > gpurun_out/r2ap_ncu.log 2>&1
