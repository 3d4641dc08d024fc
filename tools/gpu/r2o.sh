# round 2, call o: predicated aggregation (agg4 + two-candidate path); NS / 1.25e7 / C5 A/B
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2o_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2o_gputest.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_tcp0.so; do
  timeout -s KILL 300 python tools/sweep.py $lib >> gpurun_out/r2o_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2o_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2o_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 >> gpurun_out/r2o_sweep.txt 2>&1
done
