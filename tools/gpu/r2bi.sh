# round 2, call bi: ncu of the C5 pruned kernel after the unit slot sums
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_pruned -s 20 -c 1 -o gpurun_out/r2bi_c5 python bench.py --workload C5 --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2bi_ncu.log 2>&1
