# round 2, call bb: same-box A/B: one-pass merge (committed) vs + smem point cache vs cache off
set -x
for r in 1 2; do
for lib in tune/libkmeans_onepass.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_nofcache.so; do
  KMEANS_LIB_OVERRIDE=$lib timeout -s KILL 300 python bench.py --workload C2 --steps 400 --warmup 10 --repeats 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2bb_c2.jsonl 2>/dev/null
  KMEANS_LIB_OVERRIDE=$lib timeout -s KILL 300 python bench.py --workload C1 --steps 400 --warmup 10 --repeats 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2bb_c1.jsonl 2>/dev/null
done
done
