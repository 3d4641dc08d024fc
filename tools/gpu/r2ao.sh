# round 2, call ao: large-K full scan final: full GPU suite, checked build subset, bench + ncu
set -x
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2ao_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ao_gpu_tests.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or ragged or ties or dominant or configs or extreme" > gpurun_out/r2ao_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ao_checked.txt
timeout -s KILL 600 python bench.py --workload C5 --no-sort --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2ao_c5_nosort.jsonl 2> gpurun_out/r2ao_c5_nosort.err
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k "regex:k_assign_large|k_accum_large" -s 6 -c 2 -o gpurun_out/r2ao_large python bench.py --workload C5 --no-sort --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/r2ao_ncu.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2ao_launches.csv python bench.py --workload C5 --no-sort --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/r2ao_launch.log 2>&1
