# round 2, call ba: fused small-shard kernel with the points held in smem; smem limits raised only
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "configs or full_run or fused or deterministic or paper_grid or interleaved or hand or smem_sizes or k_sweep or ragged" > gpurun_out/r2ba_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ba_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_nofcache.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_nofcache.so; do
  KMEANS_LIB_OVERRIDE=$lib timeout -s KILL 300 python bench.py --workload C2 --steps 400 --warmup 10 --repeats 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2ba_c2.jsonl 2>/dev/null
  KMEANS_LIB_OVERRIDE=$lib timeout -s KILL 300 python bench.py --workload C1 --steps 400 --warmup 10 --repeats 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2ba_c1.jsonl 2>/dev/null
  KMEANS_LIB_OVERRIDE=$lib timeout -s KILL 300 python tools/sweep.py $lib --N 2000000 --reps 200 >> gpurun_out/r2ba_sweep.txt 2>&1
done
