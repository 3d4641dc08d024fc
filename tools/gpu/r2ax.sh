# round 2, call ax: e2e create / destroy timelines (pinned state blocks cached)
set -x
KMEANS_TRACE=1 timeout -s KILL 600 python tools/e2e_profile.py --workload C5 --reps 2 > gpurun_out/r2ax_e2e_c5.txt 2>&1
KMEANS_TRACE=1 timeout -s KILL 600 python tools/e2e_profile.py --workload NS --reps 2 > gpurun_out/r2ax_e2e_ns.txt 2>&1
timeout -s KILL 600 python bench.py --workload C5 --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline --no-fullscan-roofline --e2e-steps 2 > gpurun_out/r2ax_bench_c5.json 2> gpurun_out/r2ax_bench_c5.err
timeout -s KILL 600 python bench.py --steps 200 --warmup 10 --repeats 1 --no-cpu-baseline --no-fullscan-roofline --e2e-steps 2 > gpurun_out/r2ax_bench_ns.json 2> gpurun_out/r2ax_bench_ns.err
