# round 2, call bn: ncu of the large-K row merge (k_merge_sparse) at C5
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_merge_sparse -s 5 -c 1 -o gpurun_out/r2bn_merge python bench.py --workload C5 --steps 5 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2bn_ncu.log 2>&1
