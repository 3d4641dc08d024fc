# round 2, call ak: k_assign_large with rank-tree label groups
set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or extreme or configs or deterministic or dominant or full_run or fake_sharding" > gpurun_out/r2ak_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ak_tests.txt
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --no-sort --reps 5 --iters 2 >> gpurun_out/r2ak_sweep.txt 2>&1
for K in 17 32 64 128 200 400 600; do
timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --no-sort --K $K --N 20000000 --reps 10 --iters 2 >> gpurun_out/r2ak_sweep.txt 2>&1
done
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_assign_large -s 3 -c 1 -o gpurun_out/r2ak_k64 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --no-sort --K 64 --N 20000000 --reps 2 --iters 2 > gpurun_out/r2ak_ncu64.log 2>&1
