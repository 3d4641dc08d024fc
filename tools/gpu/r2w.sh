# round 2, call w: NCCL bounded wait / abort test; L2 keep re-check with the Hilbert order
set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "nccl" > gpurun_out/r2w_nccl.txt 2>&1; echo "rc=$?" >> gpurun_out/r2w_nccl.txt
for mb in 0 40 60 80 100; do
  KMEANS_L2_KEEP_MB=$mb timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N 12500000 >> gpurun_out/r2w_keep.txt 2>&1
  KMEANS_L2_KEEP_MB=$mb timeout -s KILL 300 python tools/sweep.py paper_2405_12052_b200/libkmeans.so --N 25000000 >> gpurun_out/r2w_keep.txt 2>&1
done
