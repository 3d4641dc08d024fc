# round 2, call p: per-lane run accumulators (KM_RUN_ACC) vs a butterfly per tile slot
set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/r2p_gputest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2p_gputest.txt
KMEANS_LIB_OVERRIDE=tune/libkmeans_checked.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy or large_k or k_sweep or C5 or ties" > gpurun_out/r2p_checked.txt 2>&1; echo "rc=$?" >> gpurun_out/r2p_checked.txt
for lib in paper_2405_12052_b200/libkmeans.so tune/libkmeans_run0.so; do
  timeout -s KILL 300 python tools/sweep.py $lib --workload C5 >> gpurun_out/r2p_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib --N 12500000 >> gpurun_out/r2p_sweep.txt 2>&1
  timeout -s KILL 300 python tools/sweep.py $lib >> gpurun_out/r2p_sweep.txt 2>&1
done
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "full_size_c5" > gpurun_out/r2p_c5full.txt 2>&1; echo "rc=$?" >> gpurun_out/r2p_c5full.txt
