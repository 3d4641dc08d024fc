# round 2, call ca: heavy chunks one block per tile (k_assign_heavy_tiles) vs per chunk
set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or C5 or ties or heavy or large_k or configs or dominant or deterministic or ragged" > gpurun_out/r2ca_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ca_tests.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_htold.so paper_2405_12052_b200/libkmeans.so tune/libkmeans_htold.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2ca_sweep.txt 2>&1
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_assign|k_prune|k_merge' -c 60 --csv --log-file gpurun_out/r2ca_launches.csv python bench.py --workload C5 --steps 10 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-fullscan-roofline > gpurun_out/r2ca_ncu.log 2>&1
