# round 2, call cb: ncu --set full of k_assign_heavy_tiles at C5
set -x
timeout -s KILL 300 python bench.py --workload C5 --steps 5 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2cb_plain.txt 2>&1 && \
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_heavy_tiles -s 5 -c 1 -o gpurun_out/r2cb_heavy python bench.py --workload C5 --steps 5 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2cb_ncu.log 2>&1
