# round 2, call au: C5 pruned kernel SASS breakdown + refreshed C5 bench line
set -x
timeout -s KILL 600 python bench.py --workload C5 --steps 200 --warmup 10 > gpurun_out/r2au_bench_c5.jsonl 2> gpurun_out/r2au_bench_c5.err
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_pruned -s 20 -c 1 -o gpurun_out/r2au_c5 python bench.py --workload C5 --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2au_ncu.log 2>&1
