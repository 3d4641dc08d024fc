# round 2, call s: Hilbert vs Z-curve point order (candidates per chunk, heavy chunks, time)
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2s_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2s_gputest.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_zcurve.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2s_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib >> gpurun_out/r2s_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2s_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 >> gpurun_out/r2s_sweep.txt 2>&1
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_c5_launches.csv python tools/sweep.py paper_2405_12052_b200/libkmeans.so --workload C5 --reps 5 --iters 3 > gpurun_out/r2s_launch.log 2>&1
