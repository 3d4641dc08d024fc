# round 2, call v: NS launch list + ncu of the dominant kernel (sorted path)
set -x
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2v_ns_launches.csv python bench.py --steps 20 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2v_ncu_launch.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_pruned -s 30 -c 1 -o gpurun_out/r2v_ns_pruned python bench.py --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2v_ncu_ns.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_chunk -s 5 -c 1 -o gpurun_out/r2v_ns_fullscan python bench.py --steps 5 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-sort --no-fullscan-roofline > gpurun_out/r2v_ncu_fs.log 2>&1
