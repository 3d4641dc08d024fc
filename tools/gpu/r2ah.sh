# round 2, call ah: tiled FMNMX3 large-K full scan (k_assign_large)
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or configs or ragged or ties or extreme or bisector or deterministic or full_run or fake_sharding" > gpurun_out/r2ah_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ah_tests.txt
timeout -s KILL 600 python bench.py --workload C5 --no-sort --steps 3 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/r2ah_c5_nosort.jsonl 2> gpurun_out/r2ah_c5_nosort.err
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_assign_large -s 3 -c 1 -o gpurun_out/r2ah_large python bench.py --workload C5 --no-sort --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/r2ah_ncu.log 2>&1
