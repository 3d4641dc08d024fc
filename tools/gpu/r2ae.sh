# round 2, call ae: row merge + group merge + update as one kernel (last-block ticket)
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2ae_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ae_gputest.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_mt0.so; do
  for N in 12500000 25000000 100000000; do
    timeout -s KILL 300 python tools/sweep.py $lib --N $N >> gpurun_out/r2ae_sweep.txt 2>&1
  done
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 >> gpurun_out/r2ae_sweep.txt 2>&1
done
