# round 2, call bm: heavy chunks found by k_prune, k_assign_heavy on a second stream beside k_assign_pruned
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or dominant or full_size or deterministic or ragged or profile_stages or smem_sizes" > gpurun_out/r2bm_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bm_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_nofork.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "C5 or heavy or large_k" > gpurun_out/r2bm_tests_nofork.txt 2>&1; echo "rc=$?" >> gpurun_out/r2bm_tests_nofork.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_nofork.so tune/libkmeans_base.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_nofork.so tune/libkmeans_base.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2bm_sweep.txt 2>&1
done
timeout -s KILL 600 python bench.py --workload C5 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r2bm_bench_c5.json 2> gpurun_out/r2bm_bench_c5.err
