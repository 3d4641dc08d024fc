# round 2, call ac: bisector (filtering) exclusion on top of the box test
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2ac_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ac_gputest.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_size" > gpurun_out/r2ac_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ac_checked.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_nobis.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2ac_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib >> gpurun_out/r2ac_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2ac_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --workload C3 >> gpurun_out/r2ac_sweep.txt 2>&1
done
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -k "full_size" > gpurun_out/r2ac_fullsize.txt 2>&1; echo "rc=$?" >> gpurun_out/r2ac_fullsize.txt
